// Microbenchmark (sm_100a): MUFU.SQRT / MUFU.RCP throughput alone and mixed with FFMA2, and
// the dependent-chain latency of FFMA2, FFMA, MUFU.  Times with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ float sq(float x) { float y; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rc(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// MODE 0: 16 independent MUFU.SQRT per iteration (throughput)
// MODE 1: 16 independent MUFU.RCP (each fed through an FADD: a bare rcp(rcp(x)) chain was
//         eliminated by ptxas in round 1, 0.03 cycles per "instruction")
// MODE 2: 8 MUFU + 8 FFMA2 interleaved (independent)
// MODE 3: 8 MUFU + 16 FFMA2
// MODE 4: dependent chain of FFMA2 (latency), 1 warp per SMSP
// MODE 5: dependent chain of FFMA
// MODE 6: dependent chain of MUFU.RCP
// MODE 7: dependent SHFL chain
template <int MODE>
__global__ void k(float *out, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = 1.0f + threadIdx.x * 1e-3f + i;
    float2 b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = make_float2(a[i], a[i + 8]);
    const float2 m2 = make_float2(0.999f, 0.999f), c2 = make_float2(1e-3f, 1e-3f);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = sq(a[i]) + 1.0f;
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = rc(a[i]) + 1.0f;
        } else if (MODE == 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a[i] = rc(a[i]) + 1.0f;
                b[i] = __ffma2_rn(b[i], m2, c2);
            }
        } else if (MODE == 3) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a[i] = rc(a[i]) + 1.0f;
                b[i] = __ffma2_rn(b[i], m2, c2);
                b[i] = __ffma2_rn(b[i], m2, c2);
            }
        } else if (MODE == 4) {
#pragma unroll
            for (int i = 0; i < 16; ++i) b[0] = __ffma2_rn(b[0], m2, c2);
        } else if (MODE == 5) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[0] = fmaf(a[0], 0.999f, 1e-3f);
        } else if (MODE == 6) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[0] = rc(a[0]) + 1.0f;  // MUFU + FADD latency
        } else if (MODE == 8) {  // odd warps: 16 SQRT; even warps: 64 FFMA2 (128 pipe cycles each)
            if ((threadIdx.x >> 5) & 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) a[i] = sq(a[i]) + 1.0f;
            } else {
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int i = 0; i < 8; ++i) b[i] = __ffma2_rn(b[i], m2, c2);
            }
        } else if (MODE == 9) {  // every warp: 8 SQRT + 32 FFMA2 interleaved (64 + 64 pipe cycles)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                a[i] = sq(a[i]) + 1.0f;
#pragma unroll
                for (int r = 0; r < 4; ++r) b[(i + r) & 7] = __ffma2_rn(b[(i + r) & 7], m2, c2);
            }
        } else if (MODE == 10) {  // every warp: 16 SQRT (8 of them +1 via FADD) only
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = sq(a[i]) + 1.0f;
        } else if (MODE == 7) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[0] = __shfl_down_sync(0xffffffffu, a[0], 1);
        }
    }
    float t = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) t += a[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) t += b[i].x + b[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
int run(const char *name, int blocks, int thr, int iters, double instr_per_iter, float *o) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<blocks, thr>>>(o, iters);
    CK(cudaGetLastError());
    cudaEventRecord(e0);
    k<MODE><<<blocks, thr>>>(o, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int dev, clk_khz; cudaGetDevice(&dev); cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const double warps_per_smsp = (double)blocks * thr / 32 / (148 * 4);
    const double cyc = ms * 1e-3 * 1.9e9;  // approx at ~1.9 GHz
    printf("%-34s %8.3f ms   cycles per warp-instr per SMSP (at 1.9 GHz): %.2f   (warps/SMSP %.1f)\n",
           name, ms, cyc / (warps_per_smsp * iters * instr_per_iter), warps_per_smsp);
    return 0;
}
int main() {
    float *o; CK(cudaMalloc(&o, 148 * 8 * 256 * 4));
    const int B = 148 * 4, T = 256;  // 8 warps per SMSP
    run<0>("MUFU.SQRT x16 (tput)", B, T, 4000, 16, o);
    run<1>("MUFU.RCP x16 (+FADD) (tput)", B, T, 4000, 16, o);
    run<2>("MUFU.RCP(+FADD) x8 + FFMA2 x8 (per MUFU)", B, T, 4000, 8, o);
    run<3>("MUFU.RCP(+FADD) x8 + FFMA2 x16 (per MUFU)", B, T, 4000, 8, o);
    run<8>("half warps SQRT x16 / half FFMA2 x64", B, T, 4000, 16, o);
    run<9>("SQRT x8 + FFMA2 x32 interleaved", B, T, 4000, 8, o);
    run<10>("SQRT x8 (+FADD) only", B, T, 4000, 8, o);
    run<4>("FFMA2 dep chain (latency)", 148, 32 * 4, 4000, 16, o);
    run<5>("FFMA dep chain (latency)", 148, 32 * 4, 4000, 16, o);
    run<6>("MUFU.RCP+FADD dep chain (latency)", 148, 32 * 4, 4000, 16, o);
    run<7>("SHFL dep chain (latency)", 148, 32 * 4, 4000, 16, o);
    return 0;
}
