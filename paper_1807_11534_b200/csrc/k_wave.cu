// k_wave.cu -- the temporal wavefront form of K3 (DESIGN.md §5 "wavefront"): the K-loop of a
// fixed-K solve as ONE persistent launch of blocks of KF fused iterations per strip, chained
// through progress counters in L2 instead of one launch (and one HBM round trip) per block.
//
// Same per-pixel arithmetic as k_stencil (the pipeline of k_stencil_impl.cuh, PAPER.md:119-155
// Eq. 7-9 with the rho fixed point of PAPER.md:138-141), so results are bit-identical to the
// launch-per-block form.  What changes is the schedule:
//   * a task is (block b, strip s): the warp marches every active run of the strip, so the
//     vertical dependency cone is warmed up once per run instead of once per 128-row item;
//   * consecutive blocks of a strip follow each other down the image a few rows apart, so a
//     block's input rows are read from L2 right after its producer wrote them;
//   * there is no launch boundary (ramp / tail) between blocks.
#include "k_stencil_impl.cuh"

namespace rds {

// the progress of a producer that does not exist (block 0, strips beyond the image edges)
__device__ const int32_t kWaveNone = 0x7fffffff;

template <int KF>
__global__ void __launch_bounds__(STENCIL_WARPS * 32, 2) k_wave(const WaveArgs w) {
    extern __shared__ float4 smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const StencilArgs &a = w.a;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Ctx x;
    x.pitch = a.pitch;
    x.H = a.H;
    x.tau = a.tau;
    x.theta = a.theta;
    x.inv_theta = a.inv_theta;
    x.uo = nullptr;
    x.mo = nullptr;
    x.ring = smem + warp * RING * 96 + lane;
    x.cring = smem + STENCIL_WARPS * RING * 96 + warp * CRW + lane;
    const int n_tasks = w.nblk * w.n_strips;
    WaveSlot *slot = wave_slot(x);
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(w.queue, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n_tasks) break;  // warp-uniform
        if (lane == 0) {
            const int b = t / w.n_strips, s = t - b * w.n_strips;
            const int32_t *base = w.prog + (int64_t)(b - 1) * w.n_strips;
            for (int k = 0; k < 3; ++k) {
                const int ps = s - 1 + k;
                slot->pin[k] = (b > 0 && ps >= 0 && ps < w.n_strips) ? base + ps : &kWaveNone;
            }
            slot->pout = w.prog + (int64_t)b * w.n_strips + s;
            slot->bits = w.band_bits + (int64_t)s * w.nbw;
            slot->pos = 0;
            slot->task = t;
        }
        __syncwarp();
        Wave wv;
        wv.avail = t >= w.n_strips ? 0 : a.H;
        wv.pend = wave_poll(slot);
        for (;;) {
            int pos = slot->pos, rb, re;
            if (!next_run(slot->bits, w.nbw, &pos, &rb, &re)) break;
            slot->pos = pos;
            const int tt = slot->task, b = tt / w.n_strips, s = tt - b * w.n_strips;
            const int r0 = rb * BAND_H, r1 = min(re * BAND_H, a.H);
            // rows above the run hold pinned values in both buffers: final already
            if (r0 > 0) wave_publish(x, r0);
            float acc_u = 0.0f, acc_v = 0.0f;
            // one code path per ping-pong parity (a warp vote makes the branch provably
            // uniform): each reads its plane addresses straight from the kernel parameters,
            // like k_stencil, instead of holding six more pointers in registers
            if (__all_sync(0xffffffffu, ((w.c0 + b) & 1) == 0)) {
                x.p1o = const_cast<float *>(w.p1[1]);
                x.p2o = const_cast<float *>(w.p2[1]);
                x.vo = const_cast<float *>(w.v[1]);
                run_item<KF, KF, MODE_PLAIN, true, true>(x, a, s, r0, r1, w.p1[0], w.p2[0],
                                                         w.v[0], acc_u, acc_v, wv);
            } else {
                x.p1o = const_cast<float *>(w.p1[0]);
                x.p2o = const_cast<float *>(w.p2[0]);
                x.vo = const_cast<float *>(w.v[0]);
                run_item<KF, KF, MODE_PLAIN, true, true>(x, a, s, r0, r1, w.p1[1], w.p2[1],
                                                         w.v[1], acc_u, acc_v, wv);
            }
            wave_publish(x, x.Rend);
        }
        wave_publish(x, a.H);
    }
}

typedef void (*WaveFn)(const WaveArgs);

static WaveFn wave_fn(int kf) {
    switch (kf) {
        case 4: return k_wave<4>;
        case 5: return k_wave<5>;
        case 6: return k_wave<6>;
        case 7: return k_wave<7>;
        default: return nullptr;
    }
}

bool wave_supported(int kf) { return wave_fn(kf) != nullptr; }

int wave_blocks_per_sm(int kf) {
    WaveFn fn = wave_fn(kf);
    if (!fn) return 0;
    cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         STENCIL_SMEM);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, STENCIL_WARPS * 32,
                                                      STENCIL_SMEM) != cudaSuccess)
        return 0;
    return nb;
}

cudaError_t launch_wave(int kf, const WaveArgs &w, int grid, cudaStream_t s) {
    WaveFn fn = wave_fn(kf);
    if (!fn) return cudaErrorInvalidValue;
    if (grid <= 0) return cudaSuccess;
    static bool attr[8] = {};
    if (!attr[kf]) {
        cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             STENCIL_SMEM);
        attr[kf] = true;
    }
    static const bool pdl = getenv("RDS_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(STENCIL_WARPS * 32);
    cfg.dynamicSmemBytes = STENCIL_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    void *args[] = {const_cast<WaveArgs *>(&w)};
    cudaLaunchKernelExC(&cfg, (const void *)fn, args);
    return cudaGetLastError();
}

}  // namespace rds
