// Kernel instantiation for stations with up to 16 ports.
#define VY_DEFINE_LAUNCHERS
#include "vy_launch.cuh"

namespace vy {
VY_INSTANTIATE(16)
}  // namespace vy
