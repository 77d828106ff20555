// k_stencil.cu -- dispatch of K3 (the stencil kernel template lives in k_stencil_impl.cuh,
// its instantiations in k_stencil_kf<K>.cu): kernel lookup by (k_fuse, stages, mode,
// alignment), occupancy, launch.
#include <stdlib.h>

#include "k_stencil_impl.cuh"

namespace rds {

// ---------------------------------------------------------------------------------------
// dispatch over (KF, S, MODE, ALIGNED)
// ---------------------------------------------------------------------------------------
#ifndef RDS_KF_LIST
#define RDS_KF_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)
#endif

static const int kKfMax = STENCIL_KF_MAX;

static StencilFn lookup(int kf, int stages, int mode, bool aligned, bool pro = false) {
    static StencilFn table[kKfMax + 1][kKfMax + 1][3][2];
    static StencilFn ptable[kKfMax + 1][kKfMax + 1][2];
    static bool init = false;
    if (!init) {
#define RDS_FILL(K) stencil_fill_kf##K(table[K], ptable[K]);
        RDS_KF_LIST(RDS_FILL)
#undef RDS_FILL
        auto attr = [](StencilFn f) {
            if (f)
                cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     STENCIL_SMEM);
        };
        for (auto &a : table)
            for (auto &b : a)
                for (auto &c : b)
                    for (StencilFn f : c) attr(f);
        for (auto &a : ptable)
            for (auto &b : a)
                for (StencilFn f : b) attr(f);
        init = true;
    }
    if (kf < 1 || kf > kKfMax || stages < 1 || stages > kf || mode < 0 || mode > 2)
        return nullptr;
    if (pro && mode == MODE_PLAIN) return ptable[kf][stages][aligned ? 1 : 0];
    return table[kf][stages][mode][aligned ? 1 : 0];
}

bool kf_supported(int kf) { return lookup(kf, 1, MODE_PLAIN, false) != nullptr; }

int kf_list(int32_t *out, int cap) {
    int n = 0;
    for (int k = 1; k <= kKfMax; ++k)
        if (kf_supported(k)) {
            if (n < cap && out) out[n] = k;
            ++n;
        }
    return n;
}

int stencil_blocks_per_sm(int kf, int stages, bool aligned) {
    StencilFn fn = lookup(kf, stages, MODE_PLAIN, aligned);
    if (!fn) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, STENCIL_WARPS * 32,
                                                      STENCIL_SMEM) != cudaSuccess)
        return 0;
    return nb;
}

// Warp-specialised stage chains (k_stencil_ws.cu) for the full-depth iterating launches
// (RDS_OPT_WS), where an instantiation exists.
static bool ws_on(int kf, int stages, int mode, bool aligned, bool ws) {
    return ws && mode == MODE_PLAIN && aligned && stages == kf && ws_available(stages);
}

static int n_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 1;
    }
    return n;
}

int stencil_workers_per_sm(int kf, bool aligned, bool ws) {
    if (ws_on(kf, kf, MODE_PLAIN, aligned, ws)) return ws_blocks_per_sm(kf);
    return stencil_blocks_per_sm(kf, kf, aligned) * STENCIL_WARPS;
}

cudaError_t launch_stencil(int kf, int stages, int mode, const StencilArgs &a, int grid,
                           cudaStream_t s) {
    if (ws_on(kf, stages, mode, (a.img_w & 3) == 0, a.ws != 0)) {
        // one item per CTA at a time: as many CTAs as the caller's warps had items
        int g = n_sms() * ws_blocks_per_sm(stages);
        if (g > grid * STENCIL_WARPS) g = grid * STENCIL_WARPS;
        return launch_stencil_ws(stages, a, g, s);
    }
    // the packed path needs every image-last column at lane position 3 of a quad; the prologue
    // form where the caller asks for it (a.pro, RDS_OPT_PROLOGUE)
    StencilFn fn = lookup(kf, stages, mode, (a.img_w & 3) == 0, a.pro != 0);
    if (!fn) return cudaErrorInvalidValue;
    if (grid <= 0) return cudaSuccess;
    // Programmatic dependent launch: the next stencil launch of the K loop is set up while the
    // previous one drains its last items (its CTAs take SM slots as the previous CTAs exit and
    // wait in griddepcontrol.wait until that grid has completed and its writes are visible).
    // In a captured graph this becomes a programmatic edge.  RDS_NO_PDL=1 disables it (A/B).
    static const bool pdl = getenv("RDS_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(STENCIL_WARPS * 32);
    cfg.dynamicSmemBytes = STENCIL_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void *args[] = {const_cast<StencilArgs *>(&a)};
    cudaLaunchKernelExC(&cfg, (const void *)fn, args);
    return cudaGetLastError();
}

}  // namespace rds
