// render_d6.cu -- instantiations of the render kernel for D = 6.
#include "render_kernel.cuh"

namespace sphray_b200 {
#ifndef SPHRAY_FAST_BUILD
SPHRAY_INSTANTIATE(6, 1)
SPHRAY_INSTANTIATE(6, 2)
SPHRAY_INSTANTIATE(6, 3)
SPHRAY_INSTANTIATE(6, 4)
#endif
}  // namespace sphray_b200
