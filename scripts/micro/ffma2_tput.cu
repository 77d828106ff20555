// Microbenchmark: issue throughput of scalar FFMA/FADD vs packed FFMA2/FADD2 (f32x2) and
// MUFU on sm_100a.  Each thread runs 8 independent chains; grid = 148 x 4 blocks x 256 thr.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
    u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
template <int MODE>
__global__ void k(float *out, int iters, float s) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    const float b = s, c = 1.0f - s;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // scalar FFMA, 16 independent
#pragma unroll
            for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
        } else if (MODE == 1) {  // packed FFMA2, 8 independent pairs = 16 lanes of work
            u64 bb, cc;
            asm("mov.b64 %0, {%1,%1};" : "=l"(bb) : "f"(b));
            asm("mov.b64 %0, {%1,%1};" : "=l"(cc) : "f"(c));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                u64 x; asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(a[2*i]), "f"(a[2*i+1]));
                x = ffma2(x, bb, cc);
                asm("mov.b64 {%0,%1}, %2;" : "=f"(a[2*i]), "=f"(a[2*i+1]) : "l"(x));
            }
        } else if (MODE == 2) {  // MUFU rcp, 16 independent
#pragma unroll
            for (int i = 0; i < 16; ++i) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        } else if (MODE == 3) {  // mixed: 8 FFMA2 + 4 MUFU per iteration
            u64 bb, cc;
            asm("mov.b64 %0, {%1,%1};" : "=l"(bb) : "f"(b));
            asm("mov.b64 %0, {%1,%1};" : "=l"(cc) : "f"(c));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                u64 x; asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(a[2*i]), "f"(a[2*i+1]));
                x = ffma2(x, bb, cc);
                asm("mov.b64 {%0,%1}, %2;" : "=f"(a[2*i]), "=f"(a[2*i+1]) : "l"(x));
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) asm volatile("sqrt.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        } else if (MODE == 4) {  // scalar FADD
#pragma unroll
            for (int i = 0; i < 16; ++i) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b));
        } else if (MODE == 5) {  // packed FADD2
            u64 bb; asm("mov.b64 %0, {%1,%1};" : "=l"(bb) : "f"(b));
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                u64 x; asm("mov.b64 %0, {%1,%2};" : "=l"(x) : "f"(a[2*i]), "f"(a[2*i+1]));
                x = fadd2(x, bb);
                asm("mov.b64 {%0,%1}, %2;" : "=f"(a[2*i]), "=f"(a[2*i+1]) : "l"(x));
            }
        }
    }
    float t = 0; 
#pragma unroll
    for (int i = 0; i < 16; ++i) t += a[i];
    if (t == 123.456f) out[0] = t;
}
int main() {
    float *o; cudaMalloc(&o, 4);
    int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int iters = 20000, thr = 256, blocks = sms * 4;
    const char *names[] = {"FFMA x16", "FFMA2 x8 (16 lanes)", "MUFU.RCP x16", "FFMA2 x8 + MUFU.SQRT x4", "FADD x16", "FADD2 x8"};
    const double instr_per_iter[] = {16, 8, 16, 12, 16, 8};
    for (int m = 0; m < 6; ++m) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (m) {
                case 0: k<0><<<blocks, thr>>>(o, iters, 0.5f); break;
                case 1: k<1><<<blocks, thr>>>(o, iters, 0.5f); break;
                case 2: k<2><<<blocks, thr>>>(o, iters, 0.5f); break;
                case 3: k<3><<<blocks, thr>>>(o, iters, 0.5f); break;
                case 4: k<4><<<blocks, thr>>>(o, iters, 0.5f); break;
                case 5: k<5><<<blocks, thr>>>(o, iters, 0.5f); break;
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double warp_instr = (double)blocks * thr / 32 * iters * instr_per_iter[m];
        double per_smsp_per_s = warp_instr / (sms * 4) / (ms * 1e-3);
        printf("%-26s %8.3f ms  %.3f warp-instr/ns/SMSP  (lanes-ops: %.1f T/s)\n", names[m], ms,
               per_smsp_per_s * 1e-9, (double)blocks * thr * iters * 16 / (ms * 1e-3) * 1e-12);
    }
    printf("clock attr %d kHz, err=%s\n", clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
