// Kernel instantiation for stations with up to 8 ports.
#define VY_DEFINE_LAUNCHERS
#include "vy_launch.cuh"

namespace vy {
VY_INSTANTIATE(8)
}  // namespace vy
