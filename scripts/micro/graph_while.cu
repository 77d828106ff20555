#include <cuda_runtime.h>
#include <cstdio>
__global__ void body_k(int *x, cudaGraphConditionalHandle h, int limit) {
    int v = atomicAdd(x, 1) + 1;
    cudaGraphSetConditional(h, v < limit ? 1 : 0);
}
int main() {
    int *x; cudaMalloc(&x, 4); cudaMemset(x, 0, 4);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    printf("handle %s\n", cudaGetErrorString(e));
    cudaGraphNodeParams p = {cudaGraphNodeTypeConditional};
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t n; e = cudaGraphAddNode(&n, g, nullptr, 0, &p);
    printf("add %s\n", cudaGetErrorString(e));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStream_t s; cudaStreamCreate(&s);
    e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("cap %s\n", cudaGetErrorString(e));
    body_k<<<1, 1, 0, s>>>(x, h, 1000);
    e = cudaStreamEndCapture(s, &body); printf("end %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ge; e = cudaGraphInstantiate(&ge, g, 0); printf("inst %s\n", cudaGetErrorString(e));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); e = cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int hx; cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost);
    printf("launch %s x=%d  %.3f ms (%.2f us/iter)\n", cudaGetErrorString(e), hx, ms, ms * 1000 / hx);
}
