// k_loop.cu -- the K-loop of a fixed-K solve as ONE persistent launch of K3 (DESIGN.md §5
// "persistent K-loop"): the blocks of k_fuse fused iterations that the launch-per-block form
// runs as separate kernels run here back to back inside one cooperative grid, separated by a
// grid barrier (or, when the grid is one thread-block cluster, the hardware cluster barrier).
//
// Small and mid-size images are bound by per-launch latency, not by the stencil: a 128 x 128
// image (the paper's size) marches 20 rows per item in ~3 us but pays a kernel
// launch per block.  Inside one launch a block costs the march plus one barrier.  Every item of
// every block runs run_item() of k_stencil_impl.cuh -- the same per-pixel operations -- so the
// results are bit-identical to the launch-per-block form.
#include "k_stencil_impl.cuh"

namespace rds {

namespace {

__device__ __forceinline__ void loop_grid_barrier(unsigned long long *bar, unsigned long long k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned long long target = k * gridDim.x;
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ void loop_cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace

template <int KF, bool CLUSTER>
__global__ void __launch_bounds__(STENCIL_WARPS * 32, 2) k_loop(const LoopArgs L) {
    extern __shared__ float4 smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const StencilArgs &a = L.a;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_items = *a.n_items;
    Ctx x;
    x.pitch = a.pitch;
    x.H = a.H;
    x.tau = a.tau;
    x.theta = a.theta;
    x.inv_theta = a.inv_theta;
    x.uo = a.u_out;
    x.mo = a.mask_out;
    x.chk_r0 = 0;
    x.chk_r1 = 0;
    x.ring = smem + warp * RING * 96 + lane;
    x.cring = smem + STENCIL_WARPS * RING * 96 + warp * CRW + lane;
    Wave wv{};
    for (int b = 0; b < L.nblk; ++b) {
        const int in = (L.c0 + b) & 1, out = in ^ 1;
        x.p1o = const_cast<float *>(L.p1[out]);
        x.p2o = const_cast<float *>(L.p2[out]);
        x.vo = const_cast<float *>(L.v[out]);
        const bool last = b == L.nblk - 1;
        for (;;) {
            int it = 0;
            if (lane == 0) it = atomicAdd(L.queue + b, 1);
            it = __shfl_sync(0xffffffffu, it, 0);
            if (it >= n_items) break;  // warp-uniform
            const Item item = a.items[it];
            float acc_u = 0.0f, acc_v = 0.0f;
            if (last)  // the last block also writes u and the mask
                run_item<KF, KF, MODE_WRITE_U, true, false>(x, a, item.strip, item.r0, item.r1,
                                                            L.p1[in], L.p2[in], L.v[in], acc_u,
                                                            acc_v, wv);
            else
                run_item<KF, KF, MODE_PLAIN, true, false>(x, a, item.strip, item.r0, item.r1,
                                                          L.p1[in], L.p2[in], L.v[in], acc_u,
                                                          acc_v, wv);
        }
        if (!last) {
            if (CLUSTER)
                loop_cluster_barrier();
            else
                loop_grid_barrier(L.bar, (unsigned long long)(b + 1));
        }
    }
}

typedef void (*LoopFn)(const LoopArgs);

static LoopFn loop_fn(int kf, bool cluster) {
#define RDS_LOOP_CASE(K) \
    case K: return cluster ? k_loop<K, true> : k_loop<K, false>;
    switch (kf) {
        RDS_LOOP_CASE(4)
        RDS_LOOP_CASE(5)
        RDS_LOOP_CASE(6)
        RDS_LOOP_CASE(7)
        default: return nullptr;
    }
#undef RDS_LOOP_CASE
}

bool loop_supported(int kf) { return loop_fn(kf, false) != nullptr; }

int loop_blocks_per_sm(int kf) {
    LoopFn fn = loop_fn(kf, false);
    if (!fn) return 0;
    cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         STENCIL_SMEM);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, STENCIL_WARPS * 32,
                                                      STENCIL_SMEM) != cudaSuccess)
        return 0;
    return nb;
}

// grid <= 16 CTAs: one cluster (cluster barrier); else a cooperative grid (grid barrier)
cudaError_t launch_loop(int kf, const LoopArgs &L, int grid, cudaStream_t s) {
    const bool cl = grid <= 16;
    LoopFn fn = loop_fn(kf, cl);
    if (!fn) return cudaErrorInvalidValue;
    if (grid <= 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute((const void *)fn,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         STENCIL_SMEM);
    if (e == cudaSuccess && cl && grid > 8)
        e = cudaFuncSetAttribute((const void *)fn,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    if (!cl) {
        e = cudaMemsetAsync(L.bar, 0, sizeof(unsigned long long), s);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(STENCIL_WARPS * 32);
    cfg.dynamicSmemBytes = STENCIL_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (cl) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = grid;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    } else {
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {const_cast<LoopArgs *>(&L)};
    return cudaLaunchKernelExC(&cfg, (const void *)fn, args);
}

}  // namespace rds
