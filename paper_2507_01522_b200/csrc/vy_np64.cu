// Kernel instantiation for stations with up to 64 ports.
#define VY_DEFINE_LAUNCHERS
#include "vy_launch.cuh"

namespace vy {
VY_INSTANTIATE(64)
}  // namespace vy
