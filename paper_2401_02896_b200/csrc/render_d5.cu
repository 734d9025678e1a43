// render_d5.cu -- instantiations of the render kernel for D = 5.
#include "render_kernel.cuh"

namespace sphray_b200 {
#ifndef SPHRAY_FAST_BUILD
SPHRAY_INSTANTIATE(5, 1)
SPHRAY_INSTANTIATE(5, 2)
SPHRAY_INSTANTIATE(5, 3)
SPHRAY_INSTANTIATE(5, 4)
#endif
}  // namespace sphray_b200
