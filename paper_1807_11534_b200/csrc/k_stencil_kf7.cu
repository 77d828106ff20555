// k_stencil_kf7.cu -- the k_fuse = 7 instantiations of the K3 stencil (k_stencil_impl.cuh);
// one translation unit per k_fuse so the build compiles them in parallel.
#include "k_stencil_impl.cuh"

namespace rds {

void stencil_fill_kf7(StencilFn (*t)[3][2], StencilFn (*pro)[2]) {
    Table<7, 7>::fill(t, pro);
}

}  // namespace rds
