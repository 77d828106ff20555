// Exhaustive error of the two approximate MUFU ops the stencil uses (sm_100a), against the
// correctly rounded float64 result, over every positive normal float input:
//   sqrt.approx.ftz.f32 on [2^-126, 2^128)   (the argument is |grad w|^2 + |c'|)
//   rcp.approx.ftz.f32  on [1, 2^126)        (the argument is 1 + tau sqrt(.) >= 1)
// Prints the maximum relative error of each; these bound the per-step excess of |rho| over 1
// in the fp32 kernel (reading R-G1; tests/test_gpu_parity.py RHO_STEP_EXCESS).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float sq(float x) { float y; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rc(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ unsigned long long g_max[2];  // bit patterns of non-negative doubles: order = value order
__global__ void k(uint32_t lo, uint32_t hi, int op) {
    double m = 0.0;
    for (uint64_t b = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < hi;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((uint32_t)b);
        double e;
        if (op == 0) {
            const double r = sqrt((double)x);
            e = fabs((double)sq(x) - r) / r;
        } else {
            const double r = 1.0 / (double)x;
            const float y = rc(x);
            if (r < 1.1754943508222875e-38) continue;  // result below the normal range (ftz)
            e = fabs((double)y - r) / r;
        }
        m = fmax(m, e);
    }
    atomicMax(&g_max[op], (unsigned long long)__double_as_longlong(m));
}
int main() {
    const uint32_t one = 0x3f800000u, min_norm = 0x00800000u, inf = 0x7f800000u;
    const uint32_t r_hi = 0x7e800000u;  // 2^126
    unsigned long long z[2] = {0, 0};
    cudaMemcpyToSymbol(g_max, z, sizeof z);
    k<<<148 * 16, 256>>>(min_norm, inf, 0);
    k<<<148 * 16, 256>>>(one, r_hi, 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[2];
    cudaMemcpyFromSymbol(h, g_max, sizeof h);
    double d[2];
    for (int i = 0; i < 2; ++i) d[i] = *reinterpret_cast<double *>(&h[i]);
    printf("sqrt.approx.ftz.f32 over all normal x > 0: max rel error %.6e = 2^%.3f\n", d[0], log2(d[0]));
    printf("rcp.approx.ftz.f32  over all x in [1, 2^126): max rel error %.6e = 2^%.3f\n", d[1], log2(d[1]));
    return 0;
}
