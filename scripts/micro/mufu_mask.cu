// Does MUFU throughput depend on the number of active lanes?  16 independent SQRTs per
// iteration, executed under a per-lane predicate that keeps 32, 16, 8, 4 or 1 lanes active.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float sq(float x) {
    float y;
    asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__global__ void k(float *out, int iters, int keep) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = 1.0f + threadIdx.x * 1e-3f + i;
    const bool on = (threadIdx.x & 31) % keep == 0;
    for (int it = 0; it < iters; ++it) {
        if (on) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = sq(a[i]) + 1.0f;
        }
    }
    float t = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// same with a select instead of a branch: predicated MUFU (compiler emits @P MUFU)
__global__ void k2(float *out, int iters, int keep) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = 1.0f + threadIdx.x * 1e-3f + i;
    const bool on = (threadIdx.x & 31) % keep == 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float y = a[i];
            asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p sqrt.approx.ftz.f32 %0, %1; }"
                         : "+f"(y) : "f"(a[i]), "r"((int)on));
            a[i] = y + 1.0f;
        }
    }
    float t = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float *o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int variant = 0; variant < 2; ++variant)
        for (int keep : {1, 2, 4, 8, 32}) {
            for (int r = 0; r < 2; ++r) {
                cudaEventRecord(e0);
                if (variant == 0)
                    k<<<148 * 4, 256>>>(o, 4000, keep);
                else
                    k2<<<148 * 4, 256>>>(o, 4000, keep);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double instr = 148.0 * 4 * 256 / 32 * 4000 * 16;  // warp MUFU instructions
            printf("%s active lanes %2d/32: %7.3f ms  %.2f cycles per warp MUFU per SMSP\n",
                   variant ? "predicated" : "branch    ", 32 / keep, ms,
                   ms * 1e-3 * 1.9e9 / (instr / (148 * 4)));
        }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
