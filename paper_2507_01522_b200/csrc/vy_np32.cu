// Kernel instantiation for stations with up to 32 ports.
#define VY_DEFINE_LAUNCHERS
#include "vy_launch.cuh"

namespace vy {
VY_INSTANTIATE(32)
}  // namespace vy
