// render_d4.cu -- instantiations of the render kernel for D = 4.
#include "render_kernel.cuh"

namespace sphray_b200 {
#ifndef SPHRAY_FAST_BUILD
SPHRAY_INSTANTIATE(4, 1)
SPHRAY_INSTANTIATE(4, 2)
SPHRAY_INSTANTIATE(4, 3)
SPHRAY_INSTANTIATE(4, 4)
#endif
}  // namespace sphray_b200
