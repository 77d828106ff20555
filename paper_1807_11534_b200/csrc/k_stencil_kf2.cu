// k_stencil_kf2.cu -- the k_fuse = 2 instantiations of the K3 stencil (k_stencil_impl.cuh);
// one translation unit per k_fuse so the build compiles them in parallel.
#include "k_stencil_impl.cuh"

namespace rds {

void stencil_fill_kf2(StencilFn (*t)[3][2], StencilFn (*pro)[2]) {
    Table<2, 2>::fill(t, pro);
}

}  // namespace rds
