// Microbenchmark (sm_100a): read bandwidth of a working set that stays in L2 (16-64 MB) vs one
// that streams from HBM (2 GB): float4 loads (ld.global.cg, L1 bypassed like the compact RD
// kernel's state loads), every CTA sweeping the whole buffer region it owns `reps` times.
// The L2 figure is the roofline of k_rdc_iter (f3).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void rd(const float4 *__restrict__ p, size_t n, int reps, float *out) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            const float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 12345.f) out[0] = acc;  // keeps the loads
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t sizes_mb[] = {8, 16, 32, 48, 64, 96, 2048};
    float *out;
    CK(cudaMalloc(&out, 4));
    for (size_t mb : sizes_mb) {
        const size_t bytes = mb << 20, n = bytes / 16;
        float4 *p;
        CK(cudaMalloc(&p, bytes));
        CK(cudaMemset(p, 0, bytes));
        const int reps = mb >= 1024 ? 2 : (int)(4096 / mb);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        rd<<<sms * 4, 512>>>(p, n, 1, out);  // warm (fills L2)
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int t = 0; t < 5; ++t) {
            cudaEventRecord(a);
            rd<<<sms * 4, 512>>>(p, n, reps, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("working set %5zu MB: %7.2f TB/s read\n", mb, (double)bytes * reps / (best * 1e-3) / 1e12);
        cudaFree(p);
    }
    return 0;
}
