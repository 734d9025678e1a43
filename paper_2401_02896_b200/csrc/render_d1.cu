// render_d1.cu -- instantiations of the render kernel for D = 1.
#include "render_kernel.cuh"

namespace sphray_b200 {
#ifndef SPHRAY_FAST_BUILD
SPHRAY_INSTANTIATE(1, 1)
SPHRAY_INSTANTIATE(1, 2)
SPHRAY_INSTANTIATE(1, 3)
SPHRAY_INSTANTIATE(1, 4)
#endif
}  // namespace sphray_b200
