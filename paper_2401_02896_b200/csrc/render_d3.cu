// render_d3.cu -- instantiations of the render kernel for D = 3.
#include "render_kernel.cuh"

namespace sphray_b200 {
SPHRAY_INSTANTIATE(3, 2)
#ifndef SPHRAY_FAST_BUILD
SPHRAY_INSTANTIATE(3, 1)
SPHRAY_INSTANTIATE(3, 3)
SPHRAY_INSTANTIATE(3, 4)
#endif
}  // namespace sphray_b200
