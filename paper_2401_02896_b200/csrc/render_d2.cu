// render_d2.cu -- instantiations of the render kernel for D = 2.
#include "render_kernel.cuh"

namespace sphray_b200 {
#ifndef SPHRAY_FAST_BUILD
SPHRAY_INSTANTIATE(2, 1)
SPHRAY_INSTANTIATE(2, 2)
SPHRAY_INSTANTIATE(2, 3)
SPHRAY_INSTANTIATE(2, 4)
#endif
}  // namespace sphray_b200
