// rds_api.cu -- host side of librds: the C ABI declared in include/rds.h.
//
// Handles own all device state in "padded planes" (internal.h).  rds_solve enqueues, on the
// handle's stream:  K1 fused fitting/band/init -> K2 tile compaction (+ RD count) -> item
// flags -> K2 item compaction -> ceil(K/KF) launches of K3 (ping-pong buffers; the last one
// also writes u and the mask), optionally replayed from a cached CUDA graph.  No host
// synchronisation happens inside rds_solve.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>

#include <string>

#include "internal.h"
#include "rds.h"

using namespace rds;

namespace {

thread_local std::string g_last_error;

// NVTX range for profilers (nsys / ncu --nvtx): one per host phase of a solve
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Default iterations per HBM round trip (DESIGN.md §5 sweeps): 7 where HBM traffic matters
// (C2 and larger); 4 for images of <= 2^21 pixels, whose solves are bound by item latency
// (shorter warm-up and marches: C1 1.55 vs 1.99 ms per 500 iterations).
constexpr int kDefaultKF = 7, kSmallKF = 4;
constexpr int64_t kSmallPixels = int64_t(1) << 21;
static int default_kf(int64_t H, int64_t W) { return H * W <= kSmallPixels ? kSmallKF : kDefaultKF; }
// k_fuse of the temporal wavefront (k_wave.cu) when none is set: 6 (the 7-stage pipeline
// spills once the wavefront's waits are added; 6 has the same 112 output columns per strip)
constexpr int kWaveKF = 6;
// images up to this size run fixed-K solves as one persistent launch (k_loop) by default
constexpr int64_t kPersistPixels = int64_t(1) << 22;

}  // namespace

struct rds_handle {
    int64_t H = 0, W = 0;
    int64_t img_w = 0;     // columns per image: W, or the image width of a batch
    int64_t batch = 1;     // images stacked along columns (rds_create_batch)
    int64_t pitch = 0;     // elements per padded row (multiple of 32)
    int64_t rows_alloc = 0;
    int64_t plane = 0;     // elements per plane
    int64_t origin = 0;    // element offset of pixel (0,0)
    int n_sm = 148;

    // float planes (base pointers)
    float *z = nullptr, *P = nullptr, *f = nullptr, *c = nullptr, *u = nullptr;
    float *p1[2] = {nullptr, nullptr}, *p2[2] = {nullptr, nullptr}, *v[2] = {nullptr, nullptr};
    float *wv = nullptr, *wp1 = nullptr, *wp2 = nullptr;  // warm start (lazy)
    uint8_t *lab = nullptr, *mask = nullptr;
    // tiles / items
    int n_tiles = 0;
    int32_t *tile_rd = nullptr, *tile_list = nullptr, *sub_rd = nullptr;
    uint32_t *band_flag = nullptr;   // [strip][band word] active-band bitmasks
    Item *items = nullptr;           // stencil work items
    int32_t *queue = nullptr;        // per-launch work counters
    size_t band_bytes = 0, items_bytes = 0, queue_bytes = 0;
    int bps[16][16] = {};            // cached stencil CTAs per SM [kf][stages]
    int32_t *counts = nullptr;       // [0] active tiles, [1] items, [2] chunk (bands)
    long long *n_rd_dev = nullptr;
    unsigned *absmax_bits = nullptr;
    int *flag = nullptr;
    double *e_partials = nullptr, *e_out = nullptr;
    unsigned *hist = nullptr;        // radix-select histogram (rds_band_for_fraction)
    StopRecord *stop = nullptr;      // tolerance solves (rds_solve_tol)
    double *chk = nullptr;           // per-item stopping sums of a CHECK launch
    size_t chk_bytes = 0;
    bool tol_pending = false;        // a tolerance solve's outcome is still on the device
    // float64 mode (rds_solve_gt): 7 double planes f, u, v, rho1 x2, rho2 x2 in one block
    double *d64 = nullptr, *part64 = nullptr, *cmp_out = nullptr;
    uint8_t *lab64 = nullptr;
    StopRecord *stop64 = nullptr;
    unsigned long long *bar64 = nullptr;  // grid-barrier counter of k64_persist
    bool have_gt = false;
    int cur0 = 0;                    // ping-pong buffer at the start of the last solve
    float *scratch = nullptr;        // H*W natural-order staging for swizzled-plane getters

    cudaStream_t own_stream = nullptr, stream = nullptr;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};

    bool have_image = false, have_fitting = false, solved = false, warm_pending = false;
    bool image_ok = true, p_ok = true;
    float c1 = 0, c2 = 0, gamma = 0;
    float lambda = 0, theta = 0;
    int cur = 0;  // ping-pong buffer holding the latest state
    // what rds_solve_continue needs from the last solve (labels, c' and items stay in place)
    int last_kf = 0, last_max_items = 0;
    float last_tau = 0;
    int64_t e_row0 = 0, e_row1 = -1;  // rows summed by rds_energy (-1: H)
    float *rows_buf = nullptr;        // staging of rds_get/set_state_rows with host buffers
    size_t rows_bytes = 0;

    int opt_kf = 0, opt_rows = 0, opt_timing = 0, opt_skip = 1, opt_graph = 1, opt_ctas = 0;
    int opt_norm = 0;  // stopping-rule norm: 0 Euclidean over pixels, 1 RMS (R-F2)
    int opt_split = 2;    // coupled / decoupled split (1) + grouped components (2) of compact fixed-K solves (RDS_OPT_RDC_SPLIT)
    int opt_compact = 2;  // f3: 0 dense stencil, 1 compacted RD iteration, 2 auto (default; RDS_OPT_COMPACT)
    int opt_wave = 0;     // temporal wavefront for fixed-K solves: 0 off (default), 1 on, 2 auto (RDS_OPT_WAVE)
    bool wave_ok = false; // the last solve's set-up allows the wavefront (aligned, supported kf)
    int opt_resident = 2; // small images as one resident cluster: 0 off, 1 on, 2 auto (RDS_OPT_RESIDENT)
    int opt_ws = 0;       // full-depth launches on the warp-specialised stencil (RDS_OPT_WS)
    int opt_pro = 2;      // plain launches in the prologue form: 0 off, 1 on, 2 auto (RDS_OPT_PROLOGUE)
    int opt_persist = 0;  // fixed-K loop as one persistent launch: 0 off (default), 1 on, 2 auto (RDS_OPT_PERSIST)
    bool persist_ok = false;  // the last solve's set-up allows it (aligned, supported kf, size)
    unsigned long long *loop_bar = nullptr;  // grid-barrier counter of k_loop
    int resident_fit = 0; // cached cluster schedulability for (resident_G, resident_R): 1 / -1
    int resident_G = 0, resident_R = 0;
    int opt_grid = 0;     // mid-size images resident on the whole GPU: 0 off (default), 1 / 2 on (RDS_OPT_GRID)
    int grid_fit = 0;     // cached co-residency of (grid_G, grid_R): 1 / -1
    int grid_G = 0, grid_R = 0;
    unsigned long long *grid_mail = nullptr;  // k_grid's halo mailbox ({value, tag} words)
    size_t grid_mail_n = 0;
    unsigned grid_tag = 1;       // tag of the next k_grid launch's iteration 0
    int32_t *wave_prog = nullptr;  // progress counters [blocks][strips] of k_wave
    size_t wave_prog_bytes = 0;
    // compacted RD iteration (k_rdc.cu): index map, row counts/offsets, total, compact arrays
    int32_t *rdc_idx = nullptr, *rdc_row = nullptr, *rdc_tot = nullptr;
    void *rdc_buf = nullptr;
    size_t rdc_bytes = 0;
    unsigned long long *rdc_bar = nullptr;
    double *rdc_part = nullptr;       // per-CTA stopping sums of a compact tolerance solve
    rds_stats_t stats{};

    // cached CUDA graph of the K-loop
    cudaGraphExec_t graph = nullptr;
    struct Key {
        int kf, iters, cur0, max_items, check_every, norm, wave;
        float tau, theta, tol;
        bool operator==(const Key &o) const { return memcmp(this, &o, sizeof(Key)) == 0; }
    } gkey{};

    std::string err;

    float *at(float *base) const { return base + origin; }
    uint8_t *at(uint8_t *base) const { return base + origin; }
};

static int fail(rds_t *h, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) h->err = buf;
    g_last_error = buf;
    return code;
}

#define CK(h, call)                                                                       \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail((h), e_ == cudaErrorMemoryAllocation ? RDS_ENOMEM : RDS_ECUDA,    \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                        \
    } while (0)

static void free_all(rds_t *h) {
    float *fl[] = {h->z,  h->P,     h->f,     h->c,     h->u,   h->p1[0], h->p1[1],
                   h->p2[0], h->p2[1], h->v[0], h->v[1], h->wv, h->wp1,   h->wp2};
    for (float *p : fl)
        if (p) cudaFree(p);
    void *other[] = {h->lab,     h->mask,        h->tile_rd, h->tile_list, h->band_flag,
                     h->sub_rd,
                     h->items,   h->queue,       h->counts,  h->n_rd_dev,  h->absmax_bits,
                     h->flag,    h->e_partials,  h->e_out,   h->hist,    h->scratch,
                     h->stop,    h->chk,         h->d64,     h->part64,    h->cmp_out,
                     h->lab64,   h->stop64,      h->bar64,       h->rows_buf,
                     h->rdc_idx, h->rdc_row,     h->rdc_buf,   h->rdc_bar, h->rdc_part,
                     h->wave_prog, h->loop_bar, h->grid_mail};  // rdc_tot points into rdc_row
    for (void *p : other)
        if (p) cudaFree(p);
    if (h->graph) cudaGraphExecDestroy(h->graph);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    (void)cudaGetLastError();  // a failed free must not surface in an unrelated later call
}

static cudaError_t alloc_plane(rds_t *h, float **p, float frame_value) {
    cudaError_t e = cudaMalloc(p, sizeof(float) * h->plane);
    if (e != cudaSuccess) return e;
    if (frame_value == 0.0f) return cudaMemsetAsync(*p, 0, sizeof(float) * h->plane, h->stream);
    return launch_fill_frame(*p, h->plane, frame_value, h->stream);
}

extern "C" {

int rds_create(int64_t H, int64_t W, rds_t **out) {
    if (!out) return fail(nullptr, RDS_EINVAL, "rds_create: out is NULL");
    *out = nullptr;
    if (H < 1 || W < 1) return fail(nullptr, RDS_EINVAL, "rds_create: H=%lld W=%lld must be >= 1",
                                    (long long)H, (long long)W);
    if (H * W > (int64_t(1) << 31) || H > (1 << 30) || W > (1 << 30))
        return fail(nullptr, RDS_EINVAL, "rds_create: image too large (H*W > 2^31)");
    rds_t *h = new (std::nothrow) rds_t();
    if (!h) return fail(nullptr, RDS_ENOMEM, "rds_create: host allocation failed");
    h->H = H;
    h->W = W;
    h->img_w = W;
    h->pitch = ((PAD_C + W + PAD_C_RIGHT) + 31) / 32 * 32;
    h->rows_alloc = H + 2 * PAD_R;
    h->plane = h->pitch * h->rows_alloc;
    h->origin = PAD_R * h->pitch + PAD_C;
    h->n_tiles = (int)(((H + TILE_H - 1) / TILE_H) * ((W + TILE_W - 1) / TILE_W));
    cudaError_t e = cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        int rc = fail(nullptr, RDS_ECUDA, "rds_create: cudaStreamCreate: %s", cudaGetErrorString(e));
        delete h;
        return rc;
    }
    h->stream = h->own_stream;
    {
        int dev = 0, nsm = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            nsm > 0)
            h->n_sm = nsm;
    }
#define A(call)                                                                        \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            int rc_ = fail(nullptr, e_ == cudaErrorMemoryAllocation ? RDS_ENOMEM : RDS_ECUDA, \
                           "rds_create: %s: %s", #call, cudaGetErrorString(e_));        \
            free_all(h);                                                               \
            delete h;                                                                  \
            return rc_;                                                                \
        }                                                                              \
    } while (0)
    A(alloc_plane(h, &h->z, 0.0f));
    A(alloc_plane(h, &h->f, 0.0f));
    A(alloc_plane(h, &h->c, INFINITY));
    A(alloc_plane(h, &h->u, 0.0f));
    for (int b = 0; b < 2; ++b) {
        A(alloc_plane(h, &h->p1[b], 0.0f));
        A(alloc_plane(h, &h->p2[b], 0.0f));
        A(alloc_plane(h, &h->v[b], 0.0f));
    }
    A(cudaMalloc(&h->lab, h->plane));
    A(cudaMemsetAsync(h->lab, 0, h->plane, h->stream));
    A(cudaMalloc(&h->mask, h->plane));
    A(cudaMemsetAsync(h->mask, 0, h->plane, h->stream));
    A(cudaMalloc(&h->tile_rd, sizeof(int32_t) * h->n_tiles));
    A(cudaMalloc(&h->sub_rd, sizeof(int32_t) * h->n_tiles * SUBTILES));
    A(cudaMalloc(&h->tile_list, sizeof(int32_t) * h->n_tiles));
    A(cudaMalloc(&h->counts, sizeof(int32_t) * 4));
    A(cudaMemsetAsync(h->counts, 0, sizeof(int32_t) * 4, h->stream));
    A(cudaMalloc(&h->n_rd_dev, sizeof(long long)));
    A(cudaMalloc(&h->absmax_bits, sizeof(unsigned)));
    A(cudaMalloc(&h->flag, sizeof(int)));
    A(cudaMalloc(&h->e_partials, sizeof(double) * ENERGY_WARPS * 7));
    A(cudaMalloc(&h->e_out, sizeof(double) * 7));
    for (auto &ev : h->ev) A(cudaEventCreate(&ev));
    A(cudaStreamSynchronize(h->stream));
#undef A
    *out = h;
    return RDS_OK;
}

int rds_create_batch(int64_t B, int64_t H, int64_t W, rds_t **out) {
    if (!out) return fail(nullptr, RDS_EINVAL, "rds_create_batch: out is NULL");
    *out = nullptr;
    if (B < 1 || H < 1 || W < 1)
        return fail(nullptr, RDS_EINVAL, "rds_create_batch: need B, H, W >= 1 (got %lld, %lld, %lld)",
                    (long long)B, (long long)H, (long long)W);
    if (B * W > (int64_t(1) << 30))
        return fail(nullptr, RDS_EINVAL, "rds_create_batch: B*W too large");
    const int rc = rds_create(H, B * W, out);
    if (rc) return rc;
    (*out)->img_w = W;
    (*out)->batch = B;
    return RDS_OK;
}

int rds_destroy(rds_t *h) {
    if (!h) return RDS_OK;
    if (h->stream) cudaStreamSynchronize(h->stream);
    free_all(h);
    delete h;
    return RDS_OK;
}

int rds_set_stream(rds_t *h, void *stream) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_set_stream: NULL handle");
    cudaStream_t s = stream ? (cudaStream_t)stream : h->own_stream;
    if (s != h->stream) {
        // order the switch: work already queued on the old stream completes first
        CK(h, cudaStreamSynchronize(h->stream));
        h->stream = s;
        if (h->graph) {
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
    }
    return RDS_OK;
}

int rds_set_option(rds_t *h, int key, int64_t value) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_set_option: NULL handle");
    switch (key) {
        case RDS_OPT_KFUSE:
            if (value != 0 && !kf_supported((int)value))
                return fail(h, RDS_EINVAL, "rds_set_option: k_fuse=%lld unsupported",
                            (long long)value);
            h->opt_kf = (int)value;
            return RDS_OK;
        case RDS_OPT_ITEM_ROWS:
            if (value < 0 || value > (1 << 20))
                return fail(h, RDS_EINVAL, "rds_set_option: item_rows=%lld", (long long)value);
            h->opt_rows = (int)value;
            return RDS_OK;
        case RDS_OPT_TIMING:
            h->opt_timing = value != 0;
            return RDS_OK;
        case RDS_OPT_SKIP:
            h->opt_skip = value != 0;
            return RDS_OK;
        case RDS_OPT_GRAPH:
            h->opt_graph = value != 0;
            return RDS_OK;
        case RDS_OPT_COMPACT:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: compact=%lld", (long long)value);
            h->opt_compact = (int)value;
            return RDS_OK;
        case RDS_OPT_RDC_SPLIT:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: rdc_split=%lld", (long long)value);
            h->opt_split = (int)value;
            return RDS_OK;
        case RDS_OPT_PROLOGUE:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: prologue=%lld", (long long)value);
            h->opt_pro = (int)value;
            if (h->graph) {
                cudaGraphExecDestroy(h->graph);
                h->graph = nullptr;
            }
            return RDS_OK;
        case RDS_OPT_WS:
            if (value < 0 || value > 1)
                return fail(h, RDS_EINVAL, "rds_set_option: ws=%lld", (long long)value);
            h->opt_ws = (int)value;
            if (h->graph) {
                cudaGraphExecDestroy(h->graph);
                h->graph = nullptr;
            }
            return RDS_OK;
        case RDS_OPT_PERSIST:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: persist=%lld", (long long)value);
            h->opt_persist = (int)value;
            if (h->graph) {
                cudaGraphExecDestroy(h->graph);
                h->graph = nullptr;
            }
            return RDS_OK;
        case RDS_OPT_RESIDENT:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: resident=%lld", (long long)value);
            h->opt_resident = (int)value;
            return RDS_OK;
        case RDS_OPT_GRID:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: grid=%lld", (long long)value);
            h->opt_grid = (int)value;
            return RDS_OK;
        case RDS_OPT_WAVE:
            if (value < 0 || value > 2)
                return fail(h, RDS_EINVAL, "rds_set_option: wave=%lld", (long long)value);
            h->opt_wave = (int)value;
            return RDS_OK;
        case RDS_OPT_STOP_NORM:
            if (value != 0 && value != 1)
                return fail(h, RDS_EINVAL, "rds_set_option: stop_norm=%lld", (long long)value);
            h->opt_norm = (int)value;
            return RDS_OK;
        case RDS_OPT_CTAS_PER_SM:
            if (value < 0 || value > 64)
                return fail(h, RDS_EINVAL, "rds_set_option: ctas_per_sm=%lld", (long long)value);
            h->opt_ctas = (int)value;
            if (h->graph) {
                cudaGraphExecDestroy(h->graph);
                h->graph = nullptr;
            }
            return RDS_OK;
        default:
            return fail(h, RDS_EINVAL, "rds_set_option: unknown key %d", key);
    }
}

// H x W staging buffer (host transfers of batch layouts and swizzled planes)
static int need_scratch(rds_t *h) {
    if (!h->scratch) CK(h, cudaMalloc(&h->scratch, sizeof(double) * h->H * h->W));
    return RDS_OK;
}

static int copy_in(rds_t *h, float *plane, const float *src, int on_device) {
    if (h->batch > 1) {  // dense (B, H, img_w) -> image b at columns [b img_w, (b+1) img_w)
        int rc = need_scratch(h);
        if (rc) return rc;
        const float *d = src;
        if (!on_device) {
            CK(h, cudaMemcpyAsync(h->scratch, src, sizeof(float) * h->H * h->W,
                                  cudaMemcpyHostToDevice, h->stream));
            d = h->scratch;
        }
        CK(h, launch_batch_copy(const_cast<float *>(d), h->at(plane), 4, h->pitch, (int)h->H,
                                (int)h->img_w, (int)h->batch, 1, 0, h->stream));
        if (!on_device) CK(h, cudaStreamSynchronize(h->stream));
        return RDS_OK;
    }
    cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(h, cudaMemcpy2DAsync(h->at(plane), sizeof(float) * h->pitch, src, sizeof(float) * h->W,
                            sizeof(float) * h->W, h->H, kind, h->stream));
    return RDS_OK;
}

static int check_finite(rds_t *h, const float *plane, bool *ok) {
    CK(h, cudaMemsetAsync(h->flag, 0, sizeof(int), h->stream));
    CK(h, launch_check_finite(h->at(const_cast<float *>(plane)), h->pitch, (int)h->H, (int)h->W,
                              h->flag, h->stream));
    int bad = 0;
    CK(h, cudaMemcpyAsync(&bad, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    *ok = bad == 0;
    return RDS_OK;
}

int rds_set_image(rds_t *h, const float *z, int on_device) {
    if (!h || !z) return fail(h, RDS_EINVAL, "rds_set_image: NULL argument");
    int rc = copy_in(h, h->z, z, on_device);
    if (rc) return rc;
    bool ok = true;
    if ((rc = check_finite(h, h->z, &ok))) return rc;
    h->image_ok = ok;
    h->have_image = true;
    if (!ok) return fail(h, RDS_EINVAL, "rds_set_image: image has non-finite values");
    return RDS_OK;
}

int rds_set_fitting(rds_t *h, float c1, float c2, float gamma, const float *P, int on_device) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_set_fitting: NULL handle");
    if (!isfinite(c1) || !isfinite(c2) || c1 == c2)
        return fail(h, RDS_EINVAL, "rds_set_fitting: need finite c1 != c2 (got %g, %g)", c1, c2);
    if (!isfinite(gamma) || gamma < 0.0f)
        return fail(h, RDS_EINVAL, "rds_set_fitting: gamma=%g must be finite and >= 0", gamma);
    if (gamma > 0.0f && !P)
        return fail(h, RDS_EINVAL, "rds_set_fitting: P is NULL but gamma > 0");
    if (gamma > 0.0f) {
        if (!h->P) {
            CK(h, alloc_plane(h, &h->P, 0.0f));
        }
        int rc = copy_in(h, h->P, P, on_device);
        if (rc) return rc;
        bool ok = true;
        if ((rc = check_finite(h, h->P, &ok))) return rc;
        h->p_ok = ok;
        if (!ok) {
            h->have_fitting = false;
            return fail(h, RDS_EINVAL, "rds_set_fitting: P has non-finite values");
        }
    }
    h->c1 = c1;
    h->c2 = c2;
    h->gamma = gamma;
    h->have_fitting = true;
    return RDS_OK;
}

int rds_set_state(rds_t *h, const float *v, const float *rho1, const float *rho2,
                  int on_device) {
    if (!h || !v || !rho1 || !rho2) return fail(h, RDS_EINVAL, "rds_set_state: NULL argument");
    if (!h->wv) {
        CK(h, alloc_plane(h, &h->wv, 0.0f));
        CK(h, alloc_plane(h, &h->wp1, 0.0f));
        CK(h, alloc_plane(h, &h->wp2, 0.0f));
    }
    int rc;
    if ((rc = copy_in(h, h->wv, v, on_device))) return rc;
    if ((rc = copy_in(h, h->wp1, rho1, on_device))) return rc;
    if ((rc = copy_in(h, h->wp2, rho2, on_device))) return rc;
    h->warm_pending = true;
    return RDS_OK;
}

int rds_fitting_absmax(rds_t *h, float *out) {
    if (!h || !out) return fail(h, RDS_EINVAL, "rds_fitting_absmax: NULL argument");
    if (!h->have_image || !h->have_fitting || !h->image_ok)
        return fail(h, RDS_ESTATE, "rds_fitting_absmax: image and fitting must be set");
    CK(h, cudaMemsetAsync(h->absmax_bits, 0, sizeof(unsigned), h->stream));
    CK(h, launch_absmax(h->at(h->z), h->gamma != 0.0f ? h->at(h->P) : nullptr, h->pitch,
                        (int)h->H, (int)h->W, h->c1, h->c2, h->gamma, h->absmax_bits, h->stream));
    unsigned bits = 0;
    CK(h, cudaMemcpyAsync(&bits, h->absmax_bits, sizeof bits, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    memcpy(out, &bits, sizeof bits);
    return RDS_OK;
}

int rds_band_for_fraction(rds_t *h, double q, float *delta_out) {
    if (!h || !delta_out) return fail(h, RDS_EINVAL, "rds_band_for_fraction: NULL argument");
    if (!(q >= 0.0 && q <= 1.0))
        return fail(h, RDS_EINVAL, "rds_band_for_fraction: q=%g must be in [0, 1]", q);
    if (!h->have_image || !h->have_fitting || !h->image_ok || !h->p_ok)
        return fail(h, RDS_ESTATE, "rds_band_for_fraction: image and fitting must be set");
    const int64_t N = h->H * h->W;
    int64_t k = (int64_t)ceil(q * (double)N);  // k = ceil(q N), evaluated in double
    if (k > N) k = N;
    if (k <= 0) {  // q = 0: q^ = 0, RD = {|f| < 0} = empty
        *delta_out = 0.0f;
        return RDS_OK;
    }
    if (!h->hist) CK(h, cudaMalloc(&h->hist, sizeof(unsigned) * 256));
    unsigned prefix = 0, mask = 0;
    int64_t rank = k;  // 1-based rank of the wanted |f| among the pixels matching prefix
    for (int shift = 24; shift >= 0; shift -= 8) {
        unsigned hh[256];
        CK(h, cudaMemsetAsync(h->hist, 0, sizeof hh, h->stream));
        CK(h, launch_abs_hist(h->at(h->z), h->gamma != 0.0f ? h->at(h->P) : nullptr, h->pitch,
                              (int)h->H, (int)h->W, h->c1, h->c2, h->gamma, prefix, mask, shift,
                              h->hist, h->stream));
        CK(h, cudaMemcpyAsync(hh, h->hist, sizeof hh, cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
        int d = 0;
        for (; d < 256; ++d) {
            if (rank <= (int64_t)hh[d]) break;
            rank -= hh[d];
        }
        if (d == 256) return fail(h, RDS_ECUDA, "rds_band_for_fraction: histogram inconsistent");
        prefix |= (unsigned)d << shift;
        mask |= 255u << shift;
    }
    float a;  // the k-th smallest |f|
    memcpy(&a, &prefix, sizeof a);
    // smallest float32 q^ with #{|f| < q^} >= k: the next float above a (ties at a join RD)
    *delta_out = nextafterf(a, INFINITY);
    return RDS_OK;
}

int rds_solve_q(rds_t *h, float lambda, float theta, float tau, double q, int32_t iters) {
    float delta = 0.0f;
    const int rc = rds_band_for_fraction(h, q, &delta);
    if (rc) return rc;
    return rds_solve(h, lambda, theta, tau, delta, iters);
}

// Resident stencil CTAs per SM for (kf, stages), cached (occupancy API).
static int blocks_per_sm(rds_t *h, int kf, int stages) {
    const bool aligned = (h->img_w & 3) == 0;
    int &slot = h->bps[kf][stages];
    if (slot <= 0) slot = stencil_blocks_per_sm(kf, stages, aligned);
    const int b = slot > 0 ? slot : 1;
    return (h->opt_ctas > 0 && h->opt_ctas < b) ? h->opt_ctas : b;
}

// The K-loop as a list of stencil launches.  Fixed-K solves: ceil(K/kf) launches of kf
// iterations (the last one shorter and writing u and the mask).  Tolerance solves
// (check_every = m > 0): the stopping rule is evaluated after iterations m, 2m, ... and K;
// each block between checks is cut into ceil(len/kf) near-equal launches (the longer ones
// last), and the launch ending at a check runs in CHECK mode (u, mask and the stopping sums)
// followed by k_stop_check.
struct LaunchPlan {
    int stages, mode, it_end;
    bool check;
};

static int make_plan(int kf, int iters, int check_every, LaunchPlan *out, int cap) {
    int n = 0;
    if (check_every <= 0) {
        int done = 0;
        while (done < iters) {
            const int st = (iters - done) >= kf ? kf : (iters - done);
            done += st;
            if (n < cap) out[n] = LaunchPlan{st, done == iters ? 1 : 0, done, false};
            ++n;
        }
        return n;
    }
    int prev = 0;
    while (prev < iters) {
        const int c = (iters - prev) > check_every ? prev + check_every : iters;
        const int len = c - prev, nl = (len + kf - 1) / kf, base = len / nl, rem = len % nl;
        int done = prev;
        for (int k = 0; k < nl; ++k) {
            const int st = base + (k >= nl - rem ? 1 : 0);
            done += st;
            const bool chk = k == nl - 1;
            if (n < cap) out[n] = LaunchPlan{st, chk ? 2 : 0, done, chk};
            ++n;
        }
        // a single-stage CHECK launch reads u^(l-1) from the u plane: the launch before it
        // (if any, and not itself a CHECK launch) must write u
        if (n - 1 < cap && out[n - 1].stages == 1 && nl >= 2 && n - 2 < cap)
            out[n - 2].mode = 1;
        prev = c;
    }
    return n;
}

struct TolParams {
    int check_every = 0;   // 0: fixed-K solve
    float tol = 0.0f;
    int max_iters = 0;     // K
    double norm_div = 1.0;
    int row0 = 0, row1 = -1;  // rows the stopping sums cover (row1 < 0: every row)
};

// Enqueue plan[0..n) on h->stream starting from ping-pong buffer `cur`, using work counters
// queue[qbase ..].  Check launches are followed by k_stop_check; in a graph loop body the
// last check also drives the loop (cond, body_iters, loop_end).
static cudaError_t enqueue_plan(rds_t *h, const LaunchPlan *plan, int n, int kf, int max_items,
                                float tau, float theta, const TolParams &tp, int qbase,
                                int cur, bool drive_loop, cudaGraphConditionalHandle cond,
                                int body_iters, int loop_end) {
    StencilArgs a{};
    a.c = h->at(h->c);
    a.u_out = h->at(h->u);
    a.mask_out = h->at(h->mask);
    a.items = h->items;
    a.n_items = h->counts + 1;
    a.pitch = h->pitch;
    a.ws = h->opt_ws;
    a.pro = h->opt_pro == 1 || (h->opt_pro == 2 && h->H * h->W <= (int64_t(1) << 22));
    a.H = (int)h->H;
    a.W = (int)h->W;
    a.img_w = (int)h->img_w;
    a.tau = tau;
    a.theta = theta;
    a.inv_theta = 1.0f / theta;
    a.stop = tp.check_every > 0 ? h->stop : nullptr;
    a.chk = h->chk;
    a.chk_r0 = tp.row0;
    a.chk_r1 = tp.row1 < 0 ? (int)h->H : tp.row1;
    int prev_it = n > 0 ? plan[0].it_end - plan[0].stages : 0, prev_l = 0;
    cudaError_t e = cudaSuccess;
    for (int l = 0; l < n && e == cudaSuccess; ++l) {
        const LaunchPlan &L = plan[l];
        a.p1_in = h->at(h->p1[cur]);
        a.p2_in = h->at(h->p2[cur]);
        a.v_in = h->at(h->v[cur]);
        a.p1_out = h->at(h->p1[cur ^ 1]);
        a.p2_out = h->at(h->p2[cur ^ 1]);
        a.v_out = h->at(h->v[cur ^ 1]);
        a.queue = h->queue + qbase + l;
        int grid = h->n_sm * blocks_per_sm(h, kf, L.stages);
        const int need = (max_items + STENCIL_WARPS - 1) / STENCIL_WARPS;
        if (grid > need) grid = need;
        e = launch_stencil(kf, L.stages, L.mode, a, grid, h->stream);
        if (e == cudaSuccess && L.check) {
            StopCheck c{};
            c.part = h->chk;
            c.n_part = h->counts + 1;
            c.norm_div = tp.norm_div;
            c.tol = tp.tol;
            c.block_iters = L.it_end - prev_it;
            c.block_launches = l + 1 - prev_l;
            c.max_iters = tp.max_iters;
            c.set_cond = drive_loop && l == n - 1;
            c.body_iters = body_iters;
            c.loop_end = loop_end;
            c.cond = cond;
            c.rec = h->stop;
            e = launch_stop_check(c, h->stream);
            prev_it = L.it_end;
            prev_l = l + 1;
        }
        cur ^= 1;
    }
    return e;
}

// Blocks of the temporal wavefront for a fixed-K solve of `iters` iterations: the remainder
// K mod kf runs first as one ordinary launch, the last kf iterations as the ordinary launch
// that writes u and the mask, and the nblk = K / kf - 1 blocks between them as ONE k_wave
// launch.  0 when the wavefront does not apply (fewer than one middle block).
static int wave_blocks(const rds_t *h, int kf, int iters, int check_every) {
    if (!h->wave_ok || check_every > 0 || kf < 1) return 0;
    const int nblk = iters / kf - 1;
    return nblk >= 1 ? nblk : 0;
}

static int wave_strips(const rds_t *h, int kf) {
    const int wv = wv_of(kf);
    return (int)((h->W + wv - 1) / wv);
}

// The wavefront K-loop (k_wave.cu): remainder launch, zeroed progress counters, the k_wave
// launch, the final u/mask launch.  Ping-pong parity is that of the ceil(K/kf)-launch plan.
static cudaError_t enqueue_wave(rds_t *h, int kf, int iters, int nblk, int max_items,
                                float tau, float theta) {
    StencilArgs a{};
    a.c = h->at(h->c);
    a.u_out = h->at(h->u);
    a.mask_out = h->at(h->mask);
    a.items = h->items;
    a.n_items = h->counts + 1;
    a.pitch = h->pitch;
    a.ws = h->opt_ws;
    a.pro = h->opt_pro == 1 || (h->opt_pro == 2 && h->H * h->W <= (int64_t(1) << 22));
    a.H = (int)h->H;
    a.W = (int)h->W;
    a.img_w = (int)h->img_w;
    a.tau = tau;
    a.theta = theta;
    a.inv_theta = 1.0f / theta;
    const int ns = wave_strips(h, kf);
    cudaError_t e = cudaMemsetAsync(h->queue, 0, sizeof(int32_t) * 3, h->stream);
    int cur = h->cur;
    auto ordinary = [&](int stages, int mode, int q) {
        a.p1_in = h->at(h->p1[cur]);
        a.p2_in = h->at(h->p2[cur]);
        a.v_in = h->at(h->v[cur]);
        a.p1_out = h->at(h->p1[cur ^ 1]);
        a.p2_out = h->at(h->p2[cur ^ 1]);
        a.v_out = h->at(h->v[cur ^ 1]);
        a.queue = h->queue + q;
        int grid = h->n_sm * blocks_per_sm(h, kf, stages);
        const int need = (max_items + STENCIL_WARPS - 1) / STENCIL_WARPS;
        if (grid > need) grid = need;
        cur ^= 1;
        return launch_stencil(kf, stages, mode, a, grid, h->stream);
    };
    const int r = iters % kf;
    if (e == cudaSuccess && r > 0) e = ordinary(r, 0, 0);  // mode 0: iterate
    if (e == cudaSuccess)
        e = cudaMemsetAsync(h->wave_prog, 0, sizeof(int32_t) * (size_t)nblk * ns, h->stream);
    if (e == cudaSuccess) {
        WaveArgs w{};
        w.a = a;
        for (int k = 0; k < 2; ++k) {
            w.p1[k] = h->at(h->p1[k]);
            w.p2[k] = h->at(h->p2[k]);
            w.v[k] = h->at(h->v[k]);
        }
        w.band_bits = h->band_flag;
        w.nbw = (int)(((h->H + BAND_H - 1) / BAND_H + 31) / 32);
        w.prog = h->wave_prog;
        w.queue = h->queue + 1;
        w.nblk = nblk;
        w.n_strips = ns;
        w.c0 = cur;
        int grid = h->n_sm * wave_blocks_per_sm(kf);
        const int need = (nblk * ns + STENCIL_WARPS - 1) / STENCIL_WARPS;
        if (grid > need) grid = need;
        e = launch_wave(kf, w, grid, h->stream);
        cur = (cur + nblk) & 1;
    }
    if (e == cudaSuccess) e = ordinary(kf, 1, 2);  // mode 1: + u and the mask
    return e;
}

// The persistent K-loop (k_loop.cu): the remainder K mod kf as one ordinary launch, then the
// K / kf full blocks in one launch with a barrier between blocks (the last writes u and the
// mask).  Ping-pong parity is that of the ceil(K/kf)-launch plan.
static cudaError_t enqueue_persist(rds_t *h, int kf, int iters, int max_items, float tau,
                                   float theta) {
    const int nblk = iters / kf, r = iters % kf;
    StencilArgs a{};
    a.c = h->at(h->c);
    a.u_out = h->at(h->u);
    a.mask_out = h->at(h->mask);
    a.items = h->items;
    a.n_items = h->counts + 1;
    a.pitch = h->pitch;
    a.ws = h->opt_ws;
    a.pro = h->opt_pro == 1 || (h->opt_pro == 2 && h->H * h->W <= (int64_t(1) << 22));
    a.H = (int)h->H;
    a.W = (int)h->W;
    a.img_w = (int)h->img_w;
    a.tau = tau;
    a.theta = theta;
    a.inv_theta = 1.0f / theta;
    cudaError_t e = cudaMemsetAsync(h->queue, 0, sizeof(int32_t) * (nblk + 1), h->stream);
    int cur = h->cur;
    if (e == cudaSuccess && r > 0) {
        a.p1_in = h->at(h->p1[cur]);
        a.p2_in = h->at(h->p2[cur]);
        a.v_in = h->at(h->v[cur]);
        a.p1_out = h->at(h->p1[cur ^ 1]);
        a.p2_out = h->at(h->p2[cur ^ 1]);
        a.v_out = h->at(h->v[cur ^ 1]);
        a.queue = h->queue + nblk;
        int grid = h->n_sm * blocks_per_sm(h, kf, r);
        const int need = (max_items + STENCIL_WARPS - 1) / STENCIL_WARPS;
        if (grid > need) grid = need;
        e = launch_stencil(kf, r, 0, a, grid, h->stream);
        cur ^= 1;
    }
    if (e == cudaSuccess) {
        LoopArgs L{};
        L.a = a;
        for (int k = 0; k < 2; ++k) {
            L.p1[k] = h->at(h->p1[k]);
            L.p2[k] = h->at(h->p2[k]);
            L.v[k] = h->at(h->v[k]);
        }
        L.queue = h->queue;
        L.bar = h->loop_bar;
        L.nblk = nblk;
        L.c0 = cur;
        int grid = h->n_sm * loop_blocks_per_sm(kf);
        const int need = (max_items + STENCIL_WARPS - 1) / STENCIL_WARPS;
        if (grid > need) grid = need;
        e = launch_loop(kf, L, grid, h->stream);
    }
    return e;
}

static bool persist_applies(const rds_t *h, int kf, int iters, int check_every) {
    return h->persist_ok && check_every <= 0 && kf >= 1 && iters / kf >= 2;
}

// Static K-loop: zero the work counters (and the stop record), then every planned launch.
// A tolerance solve enqueued this way runs its remaining launches as immediate exits.
static cudaError_t enqueue_loop(rds_t *h, int kf, int iters, int max_items, float tau,
                                float theta, const TolParams &tp) {
    if (persist_applies(h, kf, iters, tp.check_every))
        return enqueue_persist(h, kf, iters, max_items, tau, theta);
    const int nblk = wave_blocks(h, kf, iters, tp.check_every);
    if (nblk > 0) return enqueue_wave(h, kf, iters, nblk, max_items, tau, theta);
    const int launches = make_plan(kf, iters, tp.check_every, nullptr, 0);
    LaunchPlan *plan = new (std::nothrow) LaunchPlan[launches > 0 ? launches : 1];
    if (!plan) return cudaErrorMemoryAllocation;
    make_plan(kf, iters, tp.check_every, plan, launches);
    cudaError_t e = cudaMemsetAsync(h->queue, 0, sizeof(int32_t) * launches, h->stream);
    if (e == cudaSuccess && tp.check_every > 0)
        e = cudaMemsetAsync(h->stop, 0, sizeof(StopRecord), h->stream);
    if (e == cudaSuccess)
        e = enqueue_plan(h, plan, launches, kf, max_items, tau, theta, tp, 0, h->cur, false, 0,
                         0, 0);
    delete[] plan;
    return e;
}

// Tolerance solve as one CUDA graph with device-side control flow: a while node repeats a
// body of whole check blocks (two when a block has an odd number of launches, so the body
// keeps the ping-pong parity) for as long as the body's last k_stop_check says so, then a
// static tail covers the iterations past the last whole body.  Nothing runs after the rule
// fires except the tail's immediate exits.  Queue counters: body [0, body_launches), tail
// after that; the body zeroes its own at the start of every pass.
static cudaError_t capture_tol_graph(rds_t *h, int kf, int iters, int max_items, float tau,
                                     float theta, const TolParams &tp, cudaGraph_t *out) {
    const int m = tp.check_every;
    const int blk_n = make_plan(kf, m, m, nullptr, 0);
    const int body_blocks = (blk_n & 1) ? 2 : 1;
    const int body_iters = body_blocks * m;
    const int loop_end = (iters / body_iters) * body_iters;
    LaunchPlan *body = new (std::nothrow) LaunchPlan[body_blocks * blk_n];
    const int tail_n = make_plan(kf, iters - loop_end, m, nullptr, 0);
    LaunchPlan *tail = new (std::nothrow) LaunchPlan[tail_n > 0 ? tail_n : 1];
    if (!body || !tail) {
        delete[] body;
        delete[] tail;
        return cudaErrorMemoryAllocation;
    }
    make_plan(kf, body_iters, m, body, body_blocks * blk_n);
    make_plan(kf, iters - loop_end, m, tail, tail_n);
    for (int l = 0; l < tail_n; ++l) tail[l].it_end += loop_end;
    const int body_n = body_blocks * blk_n;

    cudaStream_t cap = nullptr;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle cond = 0;
    if (e == cudaSuccess)
        e = cudaGraphConditionalHandleCreate(&cond, g, loop_end > 0 ? 1 : 0,
                                             cudaGraphCondAssignDefault);
    cudaStream_t keep = h->stream;
    h->stream = cap;
    // prologue, the while node, the tail -- one capture sequence into g
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(cap, g, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->stop, 0, sizeof(StopRecord), cap);
    if (e == cudaSuccess)
        e = cudaMemsetAsync(h->queue + body_n, 0, sizeof(int32_t) * (tail_n > 0 ? tail_n : 1),
                            cap);
    cudaGraph_t body_g = nullptr;
    if (e == cudaSuccess) {
        cudaStreamCaptureStatus st;
        cudaGraph_t cg = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        e = cudaStreamGetCaptureInfo(cap, &st, nullptr, &cg, &deps, &nd);
        cudaGraphNode_t wnode = nullptr;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = cond;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        if (e == cudaSuccess) e = cudaGraphAddNode(&wnode, cg, deps, nd, &cp);
        if (e == cudaSuccess) {
            body_g = cp.conditional.phGraph_out[0];
            e = cudaStreamUpdateCaptureDependencies(cap, &wnode, 1,
                                                    cudaStreamSetCaptureDependencies);
        }
    }
    // the tail, after the loop
    if (e == cudaSuccess && tail_n > 0)
        e = enqueue_plan(h, tail, tail_n, kf, max_items, tau, theta, tp, body_n, h->cur, false,
                         0, 0, 0);
    {
        cudaGraph_t got = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(cap, &got);
        if (e == cudaSuccess) e = e2;
    }
    // the loop body, captured into the while node's graph
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(cap, body_g, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        cudaError_t e1 = cudaMemsetAsync(h->queue, 0, sizeof(int32_t) * body_n, cap);
        if (e1 == cudaSuccess)
            e1 = enqueue_plan(h, body, body_n, kf, max_items, tau, theta, tp, 0, h->cur, true,
                              cond, body_iters, loop_end);
        cudaGraph_t got = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(cap, &got);
        e = e1 != cudaSuccess ? e1 : e2;
    }
    h->stream = keep;
    if (cap) cudaStreamDestroy(cap);
    delete[] body;
    delete[] tail;
    if (e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return e;
    }
    *out = g;
    return cudaSuccess;
}

static cudaError_t grow(void **p, size_t *cap, size_t bytes) {
    if (bytes <= *cap) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

// f3: build the compacted RD state (index map in row-major RD order, packed neighbour codes,
// records (rho1, rho2, v, c') gathered from dense buffer 0).  Synchronises once to size the
// arrays.  RDS_OPT_COMPACT = 2 takes the compact path when its cost model beats the dense
// one by 10% (constants measured on B200, profiles/r01_compact_*.jsonl):
//   dense   per iteration ~ max(3 us, active-tile pixels / 1.0e12 /s)  (launch floor | K3 rate)
//   compact per iteration ~ 2 us (grid barrier) + n_rd / R, R = 1.5e11 /s while the compact
//           working set (~44 B per RD pixel) fits in L2, 1.0e11 /s beyond
// i.e. thin scattered bands (C3 up to delta ~ 0.1 max|f|: 1.26-4.8x; C4 at 0.02: 2x) and
// small images, whose dense solve is launch bound (C1: 1.3-1.45x); wider bands stay dense.
static bool compact_pays(int64_t n_rd, int64_t act_tile_px, size_t l2_bytes) {
    const double dense = fmax(3.0e-6, (double)act_tile_px / 1.0e12);
    const double rate = (double)n_rd * 44.0 < 0.8 * (double)l2_bytes ? 1.5e11 : 1.0e11;
    const double compact = 2.0e-6 + (double)n_rd / rate;
    return compact < 0.9 * dense;
}

struct CompactPlan {
    bool use = false;
    RdcSetup su{};
    RdcIter it{};
    const int32_t *iso = nullptr;  // split (fixed-K solves): the decoupled records
    int n_iso = 0;
    GrpPlan gp{};                  // split = 2: small components of the coupled records
    const int32_t *slots = nullptr, *lpos = nullptr;
    int n_grp = 0;                 // records iterated by k_rdc_grp
};
static int compact_prepare(rds_t *h, float tau, float theta, int iters, int check_every,
                           CompactPlan *cp) {
    cp->use = false;
    const int64_t npx = h->H * h->W;
    if (npx > INT32_MAX / 2) return RDS_OK;  // compact indices are int32: keep the dense path
    // small buffers; the H x W index map only once the path is taken.  Each buffer is
    // guarded by its own pointer, so a failed allocation is retried, never skipped.
    if (!h->rdc_row) CK(h, cudaMalloc(&h->rdc_row, sizeof(int32_t) * (2 * h->H + 1)));
    if (!h->rdc_bar) CK(h, cudaMalloc(&h->rdc_bar, RDC_BAR_BYTES));
    if (!h->rdc_part) CK(h, cudaMalloc(&h->rdc_part, sizeof(double) * 4 * RDC_MAX_GRID));
    h->rdc_tot = h->rdc_row + 2 * h->H;
    CK(h, launch_rdc_count(h->at(h->lab), h->pitch, (int)h->H, (int)h->W, h->rdc_row,
                           h->rdc_row + h->H, h->rdc_tot, h->stream));
    int32_t n = 0, act = 0;
    CK(h, cudaMemcpyAsync(&n, h->rdc_tot, sizeof n, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(&act, h->counts + 0, sizeof act, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (n >= (int32_t)RDC_IDX_MASK) return RDS_OK;  // packed codes hold 26-bit indices
    bool trial = false;  // auto mode: compact only if the grouping takes every coupled record
    if (h->opt_compact == 2) {
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        if (!compact_pays(n, (int64_t)act * TILE_H * TILE_W, (size_t)l2)) {
            // second chance for scattered bands: if the RD density inside the active tiles
            // predicts a band that falls apart into small components ((1 - p)^6 >= 0.3 of it
            // decoupled, p <= 0.18) and the grouped kernels' model (0.25 us + n_rd / 4e11 /s
            // per iteration, §6) is well under the dense one, build the compact form and keep
            // it only if every coupled record was grouped (else back to the dense path)
            const double apx = (double)act * TILE_H * TILE_W;
            const double p = apx > 0.0 ? (double)n / apx : 1.0;
            const double dense = fmax(3.0e-6, apx / 1.0e12);
            const double grouped = 0.25e-6 + (double)n / 4.0e11;
            trial = check_every <= 0 && h->opt_split >= 2 && n >= 4096 &&
                    pow(1.0 - p, 6.0) >= 0.3 && grouped < 0.7 * dense;
            if (!trial) return RDS_OK;
        }
    }
    if (!h->rdc_idx) CK(h, cudaMalloc(&h->rdc_idx, sizeof(int32_t) * npx));
    // records x2 (float4), packed codes (uint2), list, u; the split's coupled and decoupled
    // index lists and its per-chunk counts / offsets and total
    const size_t nn = (size_t)(n > 0 ? n : 1), nch = nn / 1024 + 2;
    void *pb = h->rdc_buf;
    // (+ the grouping's labels, counts, flags, ranks, class indices, block positions and
    // fallback list: 7 ints per record; its slots: < 2 per record + segment padding; counters)
    CK(h, grow(&pb, &h->rdc_bytes, nn * (16 * 2 + 8 + 4 + 4 + 4 + 4 + 4 * 9) +
                                       4 * (2 * nch + 1 + 4096 + 16)));
    h->rdc_buf = pb;
    float4 *rec0 = (float4 *)pb, *rec1 = rec0 + nn;
    uint2 *code = (uint2 *)(rec1 + nn);
    int32_t *list = (int32_t *)(code + nn);
    float *u = (float *)(list + nn);
    int32_t *cpl = (int32_t *)(u + nn), *iso = cpl + nn, *cnt = iso + nn, *off = cnt + nch,
            *ncpl = off + nch;
    int32_t *g_lab = ncpl + 1, *g_cnt = g_lab + nn, *g_bad = g_cnt + nn, *g_rank = g_bad + nn,
            *g_cidx = g_rank + nn, *g_lpos = g_cidx + nn, *g_fb = g_lpos + nn,
            *g_ctr = g_fb + nn, *g_slots = g_ctr + 16;
    CK(h, launch_rdc_fill(h->at(h->lab), h->pitch, (int)h->H, (int)h->W, h->rdc_row + h->H,
                          h->rdc_idx, list, h->stream));
    RdcSetup &su = cp->su;
    su = RdcSetup{};
    su.n = n;
    su.H = (int)h->H;
    su.W = (int)h->W;
    su.img_w = (int)h->img_w;
    su.pitch = h->pitch;
    su.list = list;
    su.idxmap = h->rdc_idx;
    su.code = code;
    su.rec = rec0;
    su.u = u;
    su.cplane = h->at(h->c);
    su.p1plane = h->at(h->p1[0]);
    su.p2plane = h->at(h->p2[0]);
    su.vplane = h->at(h->v[0]);
    su.uplane = h->at(h->u);
    su.mask = h->at(h->mask);
    CK(h, launch_rdc_gather(su, h->stream));
    RdcIter &it = cp->it;
    it = RdcIter{};
    it.n = n;
    it.code = code;
    it.rec[0] = rec0;
    it.rec[1] = rec1;
    it.u = u;
    it.tau = tau;
    it.theta = theta;
    it.inv_theta = 1.0f / theta;
    it.bar = h->rdc_bar;
    it.sel = nullptr;
    // split (fixed-K solves): pixels without an RD neighbour iterate independently (k_rdc_iso)
    if (check_every <= 0 && n >= 4096 && h->opt_split) {
        CK(h, launch_rdc_split(code, n, cnt, off, ncpl, cpl, iso, h->stream));
        int32_t nc = 0;
        CK(h, cudaMemcpyAsync(&nc, ncpl, sizeof nc, cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
        it.n = nc;
        it.sel = cpl;
        cp->iso = iso;
        cp->n_iso = n - nc;
        // split = 2: the coupled records' small connected components iterate inside one warp /
        // CTA each (k_rdc_grp); what is left keeps the grid barrier
        // (tried only where at least 15% of the RD pixels are decoupled: a scattered band of
        // density p has (1 - p)^6 of them, so p below about 0.27; a connected band has few,
        // its components are long runs that neither settle nor fit a CTA, and the label
        // rounds would be wasted -- C2 delta = .05: 7.6% decoupled, + 0.3 ms of setup)
        if (h->opt_split >= 2 && nc > 0 && (double)(n - nc) >= 0.15 * (double)n) {
            int rounds = 0;
            CK(h, launch_grp_label(code, cpl, nc, g_lab, g_cnt, g_bad, g_rank, g_cidx, g_ctr,
                                   &rounds, h->stream));
            cp->gp.rounds = rounds;
            int32_t ctr[12];
            CK(h, cudaMemcpyAsync(ctr, g_ctr, sizeof ctr, cudaMemcpyDeviceToHost, h->stream));
            CK(h, cudaStreamSynchronize(h->stream));
            // all or nothing: while any record keeps the grid barrier, its per-pass latency is
            // paid anyway and the barrier kernel absorbs the grouped records at no extra cost
            // (measured at C2's connected bands: grouped + barrier 1.8 ms vs 1.2 ms)
            if (ctr[11] == nc) {
                grp_layout(ctr, &cp->gp);
                cp->gp.rounds = rounds;
                CK(h, launch_grp_fill(cpl, nc, g_lab, g_cidx, g_rank, cp->gp, g_slots, g_lpos,
                                      g_fb, g_ctr, h->stream));
                cp->slots = g_slots;
                cp->lpos = g_lpos;
                cp->n_grp = ctr[11];
                it.n = nc - ctr[11];
                it.sel = g_fb;
            }
        }
    }
    if (trial && !(it.sel && it.n == 0)) return RDS_OK;  // some records need the barrier: dense
    cp->use = true;
    return RDS_OK;
}

// run the compact iteration and put the final state into dense buffer 0; a tolerance solve
// (check_every > 0) leaves its outcome in h->stop like the dense one (launches = 0: the state
// is in buffer 0 either way)
static int compact_run(rds_t *h, CompactPlan *cp, int iters, const TolParams &tp) {
    RdcIter &it = cp->it;
    it.K = iters;
    it.check_every = tp.check_every;
    it.tol = tp.tol;
    it.norm_div = tp.norm_div;
    it.part = h->rdc_part;
    it.rec_out = tp.check_every > 0 ? h->stop : nullptr;
    if (tp.check_every > 0) {
        StopRecord r{};
        if (it.n == 0) {  // nothing iterates: the first check (m or K) sees a zero residual
            r.flag = 1;
            r.iters = r.it = tp.check_every < iters ? tp.check_every : iters;
            r.converged = 1;
            r.checks = 1;
        }
        CK(h, cudaMemcpyAsync(h->stop, &r, sizeof r, cudaMemcpyHostToDevice, h->stream));
        if (it.n == 0) CK(h, cudaStreamSynchronize(h->stream));  // r lives on this stack
    }
    if (cp->n_iso > 0) CK(h, launch_rdc_iso(it, cp->iso, cp->n_iso, h->n_sm, h->stream));
    if (cp->n_grp > 0) CK(h, launch_rdc_grp(it, cp->gp, cp->slots, cp->lpos, h->stream));
    if (it.n > 0 || tp.check_every > 0 || !it.sel) CK(h, launch_rdc_iter(it, h->n_sm, h->stream));
    CK(h, launch_rdc_scatter(cp->su, it, h->stream));
    return RDS_OK;
}

static int solve_impl(rds_t *h, float lambda, float theta, float tau, float delta, int32_t iters,
                      int check_every, float tol) {
    if (!(lambda > 0.0f) || !isfinite(lambda))
        return fail(h, RDS_EINVAL, "rds_solve: lambda=%g must be finite and > 0", lambda);
    if (!(theta > 0.0f) || !isfinite(theta))
        return fail(h, RDS_EINVAL, "rds_solve: theta=%g must be finite and > 0", theta);
    if (!(tau > 0.0f) || !(tau <= 0.125f))
        return fail(h, RDS_EINVAL, "rds_solve: tau=%g must be in (0, 1/8]", tau);
    if (isnan(delta) || delta < 0.0f)
        return fail(h, RDS_EINVAL, "rds_solve: delta=%g must be >= 0 (inf allowed)", delta);
    if (iters < 0) return fail(h, RDS_EINVAL, "rds_solve: iters=%d must be >= 0", iters);
    if (!h->have_image || !h->have_fitting)
        return fail(h, RDS_ESTATE, "rds_solve: image and fitting must be set first");
    if (!h->image_ok || !h->p_ok)
        return fail(h, RDS_EINVAL, "rds_solve: image or P has non-finite values");

    // the temporal wavefront (k_wave) runs fixed-K solves when it applies: packed (aligned)
    // columns, a k_fuse it is built for, and, in auto mode, images above the small-image
    // size (where the launch-per-block form's item latency already binds less)
    const int kf_wave = h->opt_kf ? h->opt_kf : kWaveKF;
    h->wave_ok = h->opt_wave != 0 && check_every == 0 && (h->img_w & 3) == 0 &&
                 wave_supported(kf_wave) &&
                 (h->opt_wave == 1 || h->H * h->W > kSmallPixels);
    const int kf = h->wave_ok ? kf_wave : (h->opt_kf ? h->opt_kf : default_kf(h->H, h->W));
    // the persistent K-loop (k_loop) where launch latency, not the stencil, binds: images up
    // to 2^22 pixels in auto mode; packed columns and a supported k_fuse
    h->persist_ok = !h->wave_ok && h->opt_persist != 0 && (h->img_w & 3) == 0 &&
                    loop_supported(kf) &&
                    (h->opt_persist == 1 || h->H * h->W <= kPersistPixels);
    if (h->persist_ok && !h->loop_bar)
        CK(h, cudaMalloc(&h->loop_bar, sizeof(unsigned long long)));
    const int wv = wv_of(kf);
    const int n_strips = (int)((h->W + wv - 1) / wv);
    const int n_bands = (int)((h->H + BAND_H - 1) / BAND_H);
    // items are cut at ITEM_Q-row boundaries: at most one per ITEM_Q rows of every strip
    const int max_items = n_strips * (int)((h->H + ITEM_Q - 1) / ITEM_Q);
    const int fixed_chunk = h->opt_rows;  // rows (rounded up to ITEM_Q on the device)
    const int launches = make_plan(kf, iters, check_every, nullptr, 0);
    // work counters: one per launch of the static plan; a tolerance graph also needs the
    // counters of its loop body (up to two check blocks) besides those of its tail
    const int n_queue = launches + 1 + (check_every > 0 ? 2 * ((check_every + kf - 1) / kf) : 0);
    {
        void *pf = h->band_flag, *pi = h->items, *pq = h->queue;
        const bool realloc_items = sizeof(Item) * (size_t)max_items > h->items_bytes;
        const bool realloc_queue = sizeof(int32_t) * (size_t)n_queue > h->queue_bytes;
        CK(h, grow(&pf, &h->band_bytes, sizeof(uint32_t) * (size_t)n_strips * ((n_bands + 31) / 32)));
        CK(h, grow(&pi, &h->items_bytes, sizeof(Item) * (size_t)max_items));
        CK(h, grow(&pq, &h->queue_bytes, sizeof(int32_t) * (size_t)n_queue));
        h->band_flag = (uint32_t *)pf;
        h->items = (Item *)pi;
        h->queue = (int32_t *)pq;
        if (check_every > 0) {
            void *pc = h->chk;
            const bool realloc_chk = 2 * sizeof(double) * (size_t)max_items > h->chk_bytes;
            CK(h, grow(&pc, &h->chk_bytes, 2 * sizeof(double) * (size_t)max_items));
            h->chk = (double *)pc;
            if (!h->stop) CK(h, cudaMalloc(&h->stop, sizeof(StopRecord)));
            if (realloc_chk && h->graph) {
                cudaGraphExecDestroy(h->graph);
                h->graph = nullptr;
            }
        }
        bool realloc_prog = false;
        if (h->wave_ok) {
            const int nblk = wave_blocks(h, kf, iters, check_every);
            void *pp = h->wave_prog;
            realloc_prog = sizeof(int32_t) * (size_t)nblk * n_strips > h->wave_prog_bytes;
            CK(h, grow(&pp, &h->wave_prog_bytes, sizeof(int32_t) * ((size_t)nblk * n_strips + 1)));
            h->wave_prog = (int32_t *)pp;
        }
        if ((realloc_items || realloc_queue || realloc_prog) && h->graph) {
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
    }

    NvtxRange nvtx_solve(check_every > 0 ? "rds_solve_tol" : "rds_solve");
    if (h->opt_timing) CK(h, cudaEventRecord(h->ev[0], h->stream));
    SetupArgs s{};
    s.z = h->at(h->z);
    s.P = h->gamma != 0.0f ? h->at(h->P) : nullptr;
    if (h->warm_pending) {
        s.wv = h->at(h->wv);
        s.wp1 = h->at(h->wp1);
        s.wp2 = h->at(h->wp2);
    }
    s.f = h->at(h->f);
    s.c = h->at(h->c);
    s.u = h->at(h->u);
    s.v0 = h->at(h->v[0]);
    s.v1 = h->at(h->v[1]);
    s.p10 = h->at(h->p1[0]);
    s.p11 = h->at(h->p1[1]);
    s.p20 = h->at(h->p2[0]);
    s.p21 = h->at(h->p2[1]);
    s.lab = h->at(h->lab);
    s.mask = h->at(h->mask);
    s.tile_rd = h->tile_rd;
    s.sub_rd = h->sub_rd;
    s.pitch = h->pitch;
    s.H = (int)h->H;
    s.W = (int)h->W;
    s.img_w = (int)h->img_w;
    s.c1 = h->c1;
    s.c2 = h->c2;
    s.gamma = h->gamma;
    s.delta = delta;
    s.theta_lambda = theta * lambda;
    CK(h, launch_setup(s, h->stream));
    CK(h, launch_compact(h->tile_rd, h->n_tiles, h->tile_list, h->counts + 0, h->n_rd_dev,
                         h->stream));
    CK(h, launch_band_flags(h->sub_rd, (int)h->H, (int)h->W, wv, n_strips, h->opt_skip,
                            h->band_flag, h->stream));
    {
        const int slots = h->opt_ctas > 0
                              ? h->n_sm * blocks_per_sm(h, kf, kf) * STENCIL_WARPS
                              : h->n_sm * stencil_workers_per_sm(kf, (h->img_w & 3) == 0,
                                                                 h->opt_ws != 0);
        const int max_chunk = 1 << 30;
        CK(h, launch_build_items(h->band_flag, n_strips, n_bands, (int)h->H, slots, fixed_chunk,
                                 max_chunk,
                                 2 * kf + 4, h->items, h->counts, h->stream));
    }
    // small images: the whole fixed-K loop in one resident cluster (k_small.cu) when the image
    // fits one cluster's shared memory and such a cluster can be scheduled here
    SmallArgs sa{};
    bool small_use = false;
    // (ahead of the compact path's auto mode, which it beats where it fits; a forced compact
    // path, RDS_OPT_COMPACT = 1, still wins).  K1 put the initial state in both buffers; the
    // final state is written back into buffer 0.
    if (iters > 0 && check_every == 0 && h->opt_resident && h->opt_compact != 1 &&
        small_plan(h->H, h->W, &sa.G, &sa.R)) {
        sa.p1_in = h->at(h->p1[0]);
        sa.p2_in = h->at(h->p2[0]);
        sa.v_in = h->at(h->v[0]);
        sa.c = h->at(h->c);
        sa.p1_out = h->at(h->p1[0]);
        sa.p2_out = h->at(h->p2[0]);
        sa.v_out = h->at(h->v[0]);
        sa.u_out = h->at(h->u);
        sa.mask_out = h->at(h->mask);
        sa.n_rd = h->n_rd_dev;
        sa.pitch = h->pitch;
        sa.H = (int)h->H;
        sa.W = (int)h->W;
        sa.img_w = (int)h->img_w;
        sa.K = iters;
        sa.tau = tau;
        sa.theta = theta;
        sa.inv_theta = 1.0f / theta;
        if (h->resident_G != sa.G || h->resident_R != sa.R || h->resident_fit == 0) {
            h->resident_G = sa.G;
            h->resident_R = sa.R;
            h->resident_fit = small_cluster_fits(sa) ? 1 : -1;
        }
        small_use = h->resident_fit > 0;
    }

    // mid-size images: the whole fixed-K loop resident on the GPU (k_grid.cu), G <= #SM slabs
    // with L2-mailbox halos, where the small-image cluster does not apply
    GridArgs ga{};
    bool grid_use = false;
    if (iters > 0 && check_every == 0 && h->opt_grid && h->opt_compact != 1 && !small_use &&
        grid_plan(h->H, h->W, h->n_sm, &ga.G, &ga.R)) {
        ga.p1_in = h->at(h->p1[0]);
        ga.p2_in = h->at(h->p2[0]);
        ga.v_in = h->at(h->v[0]);
        ga.c = h->at(h->c);
        ga.p1_out = h->at(h->p1[0]);
        ga.p2_out = h->at(h->p2[0]);
        ga.v_out = h->at(h->v[0]);
        ga.u_out = h->at(h->u);
        ga.mask_out = h->at(h->mask);
        ga.n_rd = h->n_rd_dev;
        ga.pitch = h->pitch;
        ga.H = (int)h->H;
        ga.W = (int)h->W;
        ga.img_w = (int)h->img_w;
        ga.K = iters;
        ga.tau = tau;
        ga.theta = theta;
        ga.inv_theta = 1.0f / theta;
        if (h->grid_G != ga.G || h->grid_R != ga.R || h->grid_fit == 0) {
            h->grid_G = ga.G;
            h->grid_R = ga.R;
            h->grid_fit = grid_fits(ga) ? 1 : -1;
        }
        grid_use = h->grid_fit > 0;
        if (grid_use) {
            const size_t n = grid_mail_words(ga.G, ga.W);
            if (n > h->grid_mail_n) {
                if (h->grid_mail) cudaFree(h->grid_mail);
                h->grid_mail = nullptr;
                h->grid_mail_n = 0;
                CK(h, cudaMalloc(&h->grid_mail, sizeof(unsigned long long) * n));
                CK(h, cudaMemsetAsync(h->grid_mail, 0, sizeof(unsigned long long) * n,
                                      h->stream));
                h->grid_mail_n = n;
                h->grid_tag = 1;
            }
            if ((unsigned long long)h->grid_tag + (unsigned)iters + 1 >= (1ull << 31)) {
                // tags would wrap: start over from a cleared mailbox
                CK(h, cudaMemsetAsync(h->grid_mail, 0, sizeof(unsigned long long) * h->grid_mail_n,
                                      h->stream));
                h->grid_tag = 1;
            }
            ga.mail = h->grid_mail;
            ga.tag0 = h->grid_tag;
            h->grid_tag += (unsigned)iters + 1;
        }
    }

    CompactPlan cplan;
    if (iters > 0 && h->opt_compact && !small_use && !grid_use) {
        const int rc = compact_prepare(h, tau, theta, iters, check_every, &cplan);
        if (rc) return rc;
    }
    h->warm_pending = false;
    h->tol_pending = false;
    h->cur = 0;
    if (h->opt_timing) CK(h, cudaEventRecord(h->ev[1], h->stream));

    if (small_use) {
        NvtxRange nvtx_small("rds_solve (resident cluster)");
        CK(h, launch_small(sa, h->stream));
        h->cur0 = h->cur;  // the final state is written back into the same buffer
    } else if (grid_use) {
        NvtxRange nvtx_grid("rds_solve (resident grid)");
        CK(h, launch_grid(ga, h->stream));
        h->cur0 = h->cur;
    } else if (iters > 0 && cplan.use) {
        NvtxRange nvtx_rdc("rds_solve (compact RD)");
        TolParams tp;
        tp.check_every = check_every;
        tp.tol = tol;
        tp.max_iters = iters;
        tp.norm_div = h->opt_norm ? (double)h->H * (double)h->W : 1.0;
        const int rc = compact_run(h, &cplan, iters, tp);
        if (rc) return rc;
        h->cur0 = 0;
        if (check_every > 0) h->tol_pending = true;
    } else if (iters > 0) {
        TolParams tp;
        tp.check_every = check_every;
        tp.tol = tol;
        tp.max_iters = iters;
        tp.norm_div = h->opt_norm ? (double)h->H * (double)h->W : 1.0;
        rds_handle::Key key{kf,       iters,      h->cur, max_items, check_every,
                            h->opt_norm, (h->wave_ok ? 1 : 0) | (h->persist_ok ? 2 : 0),
                            tau,      theta,      tol};
        if (h->opt_graph && (launches > 1 || check_every > 0)) {
            if (!h->graph || !(h->gkey == key)) {
                if (h->graph) {
                    cudaGraphExecDestroy(h->graph);
                    h->graph = nullptr;
                }
                cudaGraph_t g = nullptr;
                cudaError_t e = cudaSuccess;
                if (check_every > 0) {
                    e = capture_tol_graph(h, kf, iters, max_items, tau, theta, tp, &g);
                } else {
                    cudaStream_t cap;
                    CK(h, cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
                    e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
                    if (e == cudaSuccess) {
                        cudaStream_t keep = h->stream;
                        h->stream = cap;
                        const cudaError_t e2 =
                            enqueue_loop(h, kf, iters, max_items, tau, theta, tp);
                        h->stream = keep;
                        e = cudaStreamEndCapture(cap, &g);
                        if (e == cudaSuccess) e = e2;
                    }
                    cudaStreamDestroy(cap);
                }
                if (e == cudaSuccess) e = cudaGraphInstantiate(&h->graph, g, 0);
                if (g) cudaGraphDestroy(g);
                if (e != cudaSuccess) {
                    h->graph = nullptr;
                    return fail(h, RDS_ECUDA, "rds_solve: graph capture failed: %s",
                                cudaGetErrorString(e));
                }
                h->gkey = key;
            }
            CK(h, cudaGraphLaunch(h->graph, h->stream));
        } else {
            CK(h, enqueue_loop(h, kf, iters, max_items, tau, theta, tp));
        }
        h->cur0 = h->cur;
        if (check_every > 0)
            h->tol_pending = true;  // the buffer holding the result is known on the device
        else if (launches & 1)
            h->cur ^= 1;
    }
    if (h->opt_timing) CK(h, cudaEventRecord(h->ev[2], h->stream));

    h->lambda = lambda;
    h->theta = theta;
    h->last_kf = kf;
    h->last_max_items = max_items;
    h->last_tau = tau;
    h->solved = true;
    rds_stats_t &st = h->stats;
    memset(&st, 0, sizeof st);
    st.H = h->H;
    st.W = h->W;
    st.n_tiles = h->n_tiles;
    st.n_items = (int64_t)n_strips * n_bands;
    st.iters = iters;
    st.k_fuse = kf;
    st.launches = (cplan.use || small_use || grid_use) ? 1 : launches;
    st.compact = cplan.use ? 1 : 0;
    st.rdc_decoupled = cplan.use ? cplan.n_iso : 0;
    st.rdc_grouped = cplan.use ? cplan.n_grp : 0;
    st.rdc_label_rounds = cplan.use ? cplan.gp.rounds : 0;
    if (cplan.use)
        st.launches = (cplan.it.n > 0 || !cplan.it.sel ? 1 : 0) + (cplan.n_iso > 0 ? 1 : 0) +
                      (cplan.gp.count[0] + cplan.gp.count[1] > 0) + (cplan.gp.count[2] > 0);
    st.wave = (!cplan.use && !small_use && !grid_use && wave_blocks(h, kf, iters, check_every) > 0) ? 1 : 0;
    st.resident = small_use ? 1 : grid_use ? 2 : 0;
    st.persist = (!cplan.use && !small_use && !grid_use && persist_applies(h, kf, iters, check_every)) ? 1 : 0;
    st.converged = 0;
    st.residual = -1.0f;
    st.check_every = check_every;
    st.item_rows = 0;  // filled by rds_get_stats (chosen on the device)
    st.item_cols = wv;
    st.setup_ms = st.loop_ms = -1.0f;
    return RDS_OK;
}

int rds_solve(rds_t *h, float lambda, float theta, float tau, float delta, int32_t iters) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_solve: NULL handle");
    return solve_impl(h, lambda, theta, tau, delta, iters, 0, 0.0f);
}

int rds_solve_tol(rds_t *h, float lambda, float theta, float tau, float delta, int32_t max_iters,
                  float tol, int32_t check_every) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_solve_tol: NULL handle");
    if (!(tol >= 0.0f)) return fail(h, RDS_EINVAL, "rds_solve_tol: tol=%g must be >= 0", tol);
    if (check_every < 0)
        return fail(h, RDS_EINVAL, "rds_solve_tol: check_every=%d must be >= 0", check_every);
    if (max_iters < 1)
        return fail(h, RDS_EINVAL, "rds_solve_tol: max_iters=%d must be >= 1", max_iters);
    // default: every 5th launch (C3: +4% over a fixed-K solve; every launch costs +19%,
    // profiles/r01_tol_overhead.jsonl)
    const int m = check_every > 0 ? check_every
                                  : 5 * (h->opt_kf ? h->opt_kf : default_kf(h->H, h->W));
    return solve_impl(h, lambda, theta, tau, delta, max_iters, m, tol);
}

// Bring the outcome of a tolerance solve to the host: which ping-pong buffer holds the
// stopped state, the iteration count and the residual (synchronises the stream).
static int resolve(rds_t *h) {
    if (!h->tol_pending) return RDS_OK;
    StopRecord r;
    CK(h, cudaMemcpyAsync(&r, h->stop, sizeof r, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    h->cur = h->cur0 ^ (r.launches & 1);  // compact path: launches = 0, state in buffer 0
    h->stats.iters = r.iters;
    if (!h->stats.compact) h->stats.launches = r.launches;
    h->stats.converged = r.converged;
    h->stats.residual = (float)r.residual;
    h->tol_pending = false;
    return RDS_OK;
}

// batch layout -> dense (B, H, img_w); elt 4 (float, swizzled or not) or 1 (bytes)
static int batch_out(rds_t *h, void *dst, const void *plane_origin, int elt, int swizzled,
                     int on_device) {
    int rc = need_scratch(h);
    if (rc) return rc;
    void *d = on_device ? dst : (void *)h->scratch;
    CK(h, launch_batch_copy(d, const_cast<void *>(plane_origin), elt, h->pitch, (int)h->H,
                            (int)h->img_w, (int)h->batch, 0, swizzled, h->stream));
    if (!on_device) {
        CK(h, cudaMemcpyAsync(dst, d, (size_t)elt * h->H * h->W, cudaMemcpyDeviceToHost,
                              h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
    }
    return RDS_OK;
}

static int copy_out(rds_t *h, void *dst, const void *plane_origin, size_t elt, int on_device) {
    if (h->batch > 1) return batch_out(h, dst, plane_origin, (int)elt, 0, on_device);
    cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(h, cudaMemcpy2DAsync(dst, elt * h->W, plane_origin, elt * h->pitch, elt * h->W, h->H,
                            kind, h->stream));
    if (!on_device) CK(h, cudaStreamSynchronize(h->stream));
    return RDS_OK;
}

// Getter of a quad-swizzled state plane (rho1, rho2, v; internal.h): unswizzled by a
// kernel, straight into a device destination or through a staging buffer for the host.
static int copy_out_swizzled(rds_t *h, float *dst, const float *plane_origin, int on_device) {
    if (h->batch > 1) return batch_out(h, dst, plane_origin, 4, 1, on_device);
    if (on_device) {
        CK(h, launch_unswizzle(plane_origin, h->pitch, (int)h->H, (int)h->W, dst, h->W,
                               h->stream));
        return RDS_OK;
    }
    {
        const int rc = need_scratch(h);
        if (rc) return rc;
    }
    CK(h, launch_unswizzle(plane_origin, h->pitch, (int)h->H, (int)h->W, h->scratch, h->W,
                           h->stream));
    CK(h, cudaMemcpyAsync(dst, h->scratch, sizeof(float) * h->H * h->W, cudaMemcpyDeviceToHost,
                          h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return RDS_OK;
}

#define NEED_SOLVED(name)                                                          \
    if (!h) return fail(nullptr, RDS_EINVAL, name ": NULL handle");                \
    if (!h->solved) return fail(h, RDS_ESTATE, name ": no solve has run yet");     \
    {                                                                              \
        const int rc_ = resolve(h);                                                \
        if (rc_) return rc_;                                                       \
    }

// ---- row strips (multi-GPU decomposition) -------------------------------------

int rds_solve_continue(rds_t *h, int32_t iters) {
    NEED_SOLVED("rds_solve_continue");
    if (iters < 0) return fail(h, RDS_EINVAL, "rds_solve_continue: iters=%d must be >= 0", iters);
    if (iters == 0) return RDS_OK;
    const int kf = h->last_kf;
    const int launches = make_plan(kf, iters, 0, nullptr, 0);
    {
        void *pq = h->queue;
        const bool realloc_queue = sizeof(int32_t) * (size_t)(launches + 3) > h->queue_bytes;
        CK(h, grow(&pq, &h->queue_bytes, sizeof(int32_t) * (size_t)(launches + 3)));
        h->queue = (int32_t *)pq;
        const int nblk = wave_blocks(h, kf, iters, 0);
        void *pp = h->wave_prog;
        const size_t pb = sizeof(int32_t) * ((size_t)nblk * wave_strips(h, kf) + 1);
        const bool realloc_prog = nblk > 0 && pb > h->wave_prog_bytes;
        if (nblk > 0) CK(h, grow(&pp, &h->wave_prog_bytes, pb));
        h->wave_prog = (int32_t *)pp;
        if ((realloc_queue || realloc_prog) && h->graph) {  // the cached graph points at them
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
    }
    NvtxRange nvtx("rds_solve_continue");
    if (h->opt_timing) {
        CK(h, cudaEventRecord(h->ev[0], h->stream));
        CK(h, cudaEventRecord(h->ev[1], h->stream));
    }
    TolParams tp;
    tp.max_iters = iters;
    CK(h, enqueue_loop(h, kf, iters, h->last_max_items, h->last_tau, h->theta, tp));
    if (launches & 1) h->cur ^= 1;
    if (h->opt_timing) CK(h, cudaEventRecord(h->ev[2], h->stream));
    h->stats.iters += iters;
    h->stats.launches += launches;
    h->stats.converged = 0;
    h->stats.residual = -1.0f;
    h->stats.check_every = 0;
    return RDS_OK;
}

int rds_continue_check(rds_t *h, int32_t iters, int64_t row0, int64_t row1, double *sums) {
    NEED_SOLVED("rds_continue_check");
    if (iters < 1) return fail(h, RDS_EINVAL, "rds_continue_check: iters=%d must be >= 1", iters);
    if (!sums) return fail(h, RDS_EINVAL, "rds_continue_check: NULL sums");
    if (row0 < 0 || row1 > h->H || row0 > row1)
        return fail(h, RDS_EINVAL, "rds_continue_check: rows [%lld, %lld) outside [0, %lld)",
                    (long long)row0, (long long)row1, (long long)h->H);
    if (h->tol_pending) {  // a tolerance solve's state: bring its outcome to the host first
        const int rc = resolve(h);
        if (rc) return rc;
    }
    const int kf = h->last_kf;
    const int launches = make_plan(kf, iters, iters, nullptr, 0);
    {
        void *pq = h->queue, *pc = h->chk;
        const bool realloc_queue = sizeof(int32_t) * (size_t)launches > h->queue_bytes;
        CK(h, grow(&pq, &h->queue_bytes, sizeof(int32_t) * (size_t)launches));
        h->queue = (int32_t *)pq;
        const bool realloc_chk = 2 * sizeof(double) * (size_t)h->last_max_items > h->chk_bytes;
        CK(h, grow(&pc, &h->chk_bytes, 2 * sizeof(double) * (size_t)h->last_max_items));
        h->chk = (double *)pc;
        if (!h->stop) CK(h, cudaMalloc(&h->stop, sizeof(StopRecord)));
        if ((realloc_queue || realloc_chk) && h->graph) {
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
    }
    NvtxRange nvtx("rds_continue_check");
    TolParams tp;
    tp.check_every = iters;  // one check, after the last iteration
    tp.tol = -1.0f;          // never "converged": only the sums are wanted
    tp.max_iters = iters;
    tp.row0 = (int)row0;
    tp.row1 = (int)row1;
    CK(h, enqueue_loop(h, kf, iters, h->last_max_items, h->last_tau, h->theta, tp));
    StopRecord rec{};
    CK(h, cudaMemcpyAsync(&rec, h->stop, sizeof rec, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    if (launches & 1) h->cur ^= 1;
    sums[0] = rec.su;
    sums[1] = rec.sv;
    h->stats.iters += iters;
    h->stats.launches += launches;
    return RDS_OK;
}

int rds_abs_histogram(rds_t *h, int64_t row0, int64_t row1, uint32_t prefix, uint32_t mask,
                      int32_t shift, uint32_t *out) {
    if (!h || !out) return fail(h, RDS_EINVAL, "rds_abs_histogram: NULL argument");
    if (!h->have_image || !h->have_fitting || !h->image_ok || !h->p_ok)
        return fail(h, RDS_ESTATE, "rds_abs_histogram: image and fitting must be set");
    if (row0 < 0 || row1 > h->H || row0 > row1 || (shift != 0 && shift != 8 && shift != 16 &&
                                                   shift != 24))
        return fail(h, RDS_EINVAL, "rds_abs_histogram: rows [%lld, %lld) or shift %d invalid",
                    (long long)row0, (long long)row1, shift);
    if (!h->hist) CK(h, cudaMalloc(&h->hist, sizeof(unsigned) * 256));
    CK(h, cudaMemsetAsync(h->hist, 0, sizeof(unsigned) * 256, h->stream));
    if (row1 > row0)
        CK(h, launch_abs_hist(h->at(h->z) + row0 * h->pitch,
                              h->gamma != 0.0f ? h->at(h->P) + row0 * h->pitch : nullptr,
                              h->pitch, (int)(row1 - row0), (int)h->W, h->c1, h->c2, h->gamma,
                              prefix, mask, shift, h->hist, h->stream));
    CK(h, cudaMemcpyAsync(out, h->hist, sizeof(unsigned) * 256, cudaMemcpyDeviceToHost,
                          h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return RDS_OK;
}

static int state_rows(rds_t *h, int64_t row0, int64_t nrows, float *buf, int on_device,
                      int put, const char *name) {
    if (h->batch > 1) return fail(h, RDS_EINVAL, "%s: not available on a batch handle", name);
    if (row0 < 0 || nrows < 0 || row0 + nrows > h->H)
        return fail(h, RDS_EINVAL, "%s: rows [%lld, %lld) outside [0, %lld)", name,
                    (long long)row0, (long long)(row0 + nrows), (long long)h->H);
    if (nrows == 0) return RDS_OK;
    if (!buf) return fail(h, RDS_EINVAL, "%s: NULL buffer", name);
    const int64_t n = nrows * h->W;  // elements per plane
    const size_t bytes = sizeof(float) * 3 * (size_t)n;
    float *d = buf;
    if (!on_device) {
        void *pb = h->rows_buf;
        CK(h, grow(&pb, &h->rows_bytes, bytes));
        h->rows_buf = (float *)pb;
        d = h->rows_buf;
        if (put) CK(h, cudaMemcpyAsync(d, buf, bytes, cudaMemcpyHostToDevice, h->stream));
    }
    float *planes[3] = {h->v[h->cur], h->p1[h->cur], h->p2[h->cur]};
    for (int q = 0; q < 3; ++q)
        CK(h, launch_batch_copy(d + q * n, h->at(planes[q]) + row0 * h->pitch, 4, h->pitch,
                                (int)nrows, (int)h->W, 1, put, 1, h->stream));
    if (!on_device) {
        if (!put) CK(h, cudaMemcpyAsync(buf, d, bytes, cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
    }
    return RDS_OK;
}

int rds_get_state_rows(rds_t *h, int64_t row0, int64_t nrows, float *out, int on_device) {
    NEED_SOLVED("rds_get_state_rows");
    return state_rows(h, row0, nrows, out, on_device, 0, "rds_get_state_rows");
}

int rds_set_state_rows(rds_t *h, int64_t row0, int64_t nrows, const float *in, int on_device) {
    NEED_SOLVED("rds_set_state_rows");
    return state_rows(h, row0, nrows, const_cast<float *>(in), on_device, 1,
                      "rds_set_state_rows");
}

int rds_set_energy_rows(rds_t *h, int64_t row0, int64_t row1) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_set_energy_rows: NULL handle");
    if (row1 < 0) row1 = h->H;
    if (row0 < 0 || row0 > row1 || row1 > h->H)
        return fail(h, RDS_EINVAL, "rds_set_energy_rows: rows [%lld, %lld) outside [0, %lld)",
                    (long long)row0, (long long)row1, (long long)h->H);
    h->e_row0 = row0;
    h->e_row1 = row1;
    return RDS_OK;
}

int rds_get_u(rds_t *h, float *out, int on_device) {
    NEED_SOLVED("rds_get_u");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_u: NULL out");
    return copy_out(h, out, h->at(h->u), sizeof(float), on_device);
}

int rds_get_mask(rds_t *h, uint8_t *out, int on_device) {
    NEED_SOLVED("rds_get_mask");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_mask: NULL out");
    return copy_out(h, out, h->at(h->mask), 1, on_device);
}

int rds_get_v(rds_t *h, float *out, int on_device) {
    NEED_SOLVED("rds_get_v");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_v: NULL out");
    return copy_out_swizzled(h, out, h->at(h->v[h->cur]), on_device);
}

int rds_get_p(rds_t *h, float *rho1, float *rho2, int on_device) {
    NEED_SOLVED("rds_get_p");
    if (!rho1 || !rho2) return fail(h, RDS_EINVAL, "rds_get_p: NULL out");
    int rc = copy_out_swizzled(h, rho1, h->at(h->p1[h->cur]), on_device);
    if (rc) return rc;
    return copy_out_swizzled(h, rho2, h->at(h->p2[h->cur]), on_device);
}

int rds_get_fitting(rds_t *h, float *out, int on_device) {
    NEED_SOLVED("rds_get_fitting");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_fitting: NULL out");
    return copy_out(h, out, h->at(h->f), sizeof(float), on_device);
}

int rds_get_labels(rds_t *h, uint8_t *out, int on_device) {
    NEED_SOLVED("rds_get_labels");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_labels: NULL out");
    return copy_out(h, out, h->at(h->lab), 1, on_device);
}

int rds_get_active_tiles(rds_t *h, int32_t *out, int64_t cap, int64_t *count) {
    NEED_SOLVED("rds_get_active_tiles");
    if (!count) return fail(h, RDS_EINVAL, "rds_get_active_tiles: NULL count");
    int32_t n = 0;
    CK(h, cudaMemcpyAsync(&n, h->counts, sizeof n, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    *count = n;
    if (cap < n) return fail(h, RDS_EINVAL, "rds_get_active_tiles: cap %lld < count %d",
                             (long long)cap, n);
    if (n > 0) {
        if (!out) return fail(h, RDS_EINVAL, "rds_get_active_tiles: NULL out");
        CK(h, cudaMemcpyAsync(out, h->tile_list, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                              h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
    }
    return RDS_OK;
}

int rds_tile_shape(int *th, int *tw) {
    if (!th || !tw) return fail(nullptr, RDS_EINVAL, "rds_tile_shape: NULL argument");
    *th = TILE_H;
    *tw = TILE_W;
    return RDS_OK;
}

int rds_energy(rds_t *h, rds_energy_t *out) {
    NEED_SOLVED("rds_energy");
    NvtxRange nvtx_energy("rds_energy");
    if (!out) return fail(h, RDS_EINVAL, "rds_energy: NULL out");
    EnergyArgs a{};
    a.f = h->at(h->f);
    a.u = h->at(h->u);
    a.v = h->at(h->v[h->cur]);
    a.p1 = h->at(h->p1[h->cur]);
    a.p2 = h->at(h->p2[h->cur]);
    a.pitch = h->pitch;
    a.H = (int)h->H;
    a.W = (int)h->W;
    a.img_w = (int)h->img_w;
    a.row0 = (int)h->e_row0;
    a.row1 = (int)(h->e_row1 < 0 ? h->H : h->e_row1);
    a.partials = h->e_partials;
    a.out = h->e_out;
    a.lab = h->at(h->lab);
    a.lambda = h->lambda;
    a.theta = h->theta;
    CK(h, launch_energy(a, h->stream));
    double s[7];
    CK(h, cudaMemcpyAsync(s, h->e_out, sizeof s, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    const double lam = (double)h->lambda;
    out->TV_v = s[0];
    out->fit_v = lam * s[1];
    out->E_v = s[0] + lam * s[1];
    out->E_u = s[2] + lam * s[3];
    out->D_p = s[4];
    out->gap = out->E_v - out->D_p;
    out->F_rd = s[5] + s[6] / (2.0 * (double)h->theta) + lam * s[1];
    return RDS_OK;
}

int rds_get_stats(rds_t *h, rds_stats_t *out) {
    NEED_SOLVED("rds_get_stats");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_stats: NULL out");
    int32_t cnt[4];
    long long nrd = 0;
    CK(h, cudaMemcpyAsync(cnt, h->counts, sizeof cnt, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaMemcpyAsync(&nrd, h->n_rd_dev, sizeof nrd, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    h->stats.n_active_tiles = cnt[0];
    h->stats.n_active_items = cnt[1];
    h->stats.item_rows = cnt[2];
    h->stats.n_active_cells = cnt[3];
    h->stats.n_rd = nrd;
    if (h->opt_timing) {
        CK(h, cudaEventElapsedTime(&h->stats.setup_ms, h->ev[0], h->ev[1]));
        CK(h, cudaEventElapsedTime(&h->stats.loop_ms, h->ev[1], h->ev[2]));
    }
    *out = h->stats;
    return RDS_OK;
}

int rds_solve_gt(rds_t *h, float lambda, float theta, float tau, float delta,
                 int32_t max_iters, double tol, int32_t check_every, rds_gt_t *out) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_solve_gt: NULL handle");
    if (!(lambda > 0.0f) || !isfinite(lambda) || !(theta > 0.0f) || !isfinite(theta))
        return fail(h, RDS_EINVAL, "rds_solve_gt: need finite lambda, theta > 0");
    if (!(tau > 0.0f) || !(tau <= 0.125f))
        return fail(h, RDS_EINVAL, "rds_solve_gt: tau=%g must be in (0, 1/8]", tau);
    if (isnan(delta) || delta < 0.0f)
        return fail(h, RDS_EINVAL, "rds_solve_gt: delta=%g must be >= 0", delta);
    if (max_iters < 1 || check_every < 1 || !(tol >= 0.0))
        return fail(h, RDS_EINVAL, "rds_solve_gt: need max_iters >= 1, check_every >= 1, "
                                   "tol >= 0");
    if (!h->have_image || !h->have_fitting)
        return fail(h, RDS_ESTATE, "rds_solve_gt: image and fitting must be set first");
    if (!h->image_ok || !h->p_ok)
        return fail(h, RDS_EINVAL, "rds_solve_gt: image or P has non-finite values");
    NvtxRange nvtx_gt("rds_solve_gt");
    // f, u, v, rho1 x2, rho2 x2, v (second buffer): 8 double planes; every buffer guarded by
    // its own pointer (a failed allocation is retried on the next call, never skipped)
    if (!h->d64) {
        CK(h, cudaMalloc(&h->d64, sizeof(double) * h->plane * 8));
        CK(h, cudaMemsetAsync(h->d64, 0, sizeof(double) * h->plane * 8, h->stream));
    }
    if (!h->lab64) {
        CK(h, cudaMalloc(&h->lab64, h->plane));
        CK(h, cudaMemsetAsync(h->lab64, 0, h->plane, h->stream));
    }
    if (!h->part64) CK(h, cudaMalloc(&h->part64, sizeof(double) * 4 * F64P_MAX_GRID));
    if (!h->cmp_out) CK(h, cudaMalloc(&h->cmp_out, sizeof(double) * 2));
    if (!h->stop64) CK(h, cudaMalloc(&h->stop64, sizeof(StopRecord)));
    if (!h->bar64) CK(h, cudaMalloc(&h->bar64, sizeof(unsigned long long)));
    CK(h, cudaMemsetAsync(h->stop64, 0, sizeof(StopRecord), h->stream));
    F64Args a{};
    a.z = h->at(h->z);
    a.P = h->gamma != 0.0f ? h->at(h->P) : nullptr;
    double *pl[8];
    for (int k = 0; k < 8; ++k) pl[k] = h->d64 + h->plane * k + h->origin;
    a.f = pl[0];
    a.u = pl[1];
    a.v = pl[2];
    a.p1[0] = pl[3];
    a.p1[1] = pl[4];
    a.p2[0] = pl[5];
    a.p2[1] = pl[6];
    a.v2 = pl[7];
    a.lab = h->lab64 + h->origin;
    a.stop = h->stop64;
    a.pitch = h->pitch;
    a.H = (int)h->H;
    a.W = (int)h->W;
    a.img_w = (int)h->img_w;
    a.c1 = h->c1;
    a.c2 = h->c2;
    a.gamma = h->gamma;
    a.delta = delta;
    a.tau = (double)tau;
    a.theta = (double)theta;
    a.theta_lambda = (double)theta * (double)lambda;
    CK(h, launch_f64_init(a, h->stream));
    F64Persist q{};
    q.a = a;
    q.a.stop = h->stop64;
    q.v[0] = pl[2];
    q.v[1] = pl[7];
    q.max_iters = max_iters;
    q.check_every = check_every;
    q.tol = tol;
    q.norm_div = h->opt_norm ? (double)h->H * (double)h->W : 1.0;
    q.part = h->part64;
    q.bar = h->bar64;
    CK(h, launch_f64_persist(q, h->n_sm, h->stream));
    StopRecord rec{};
    CK(h, cudaMemcpyAsync(&rec, h->stop64, sizeof rec, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    h->have_gt = true;
    if (out) {
        out->iters = rec.iters;
        out->converged = rec.converged;
        out->residual = rec.residual;
    }
    return RDS_OK;
}

int rds_get_u_gt(rds_t *h, double *out, int on_device) {
    if (!h) return fail(nullptr, RDS_EINVAL, "rds_get_u_gt: NULL handle");
    if (!h->have_gt) return fail(h, RDS_ESTATE, "rds_get_u_gt: no rds_solve_gt has run yet");
    if (!out) return fail(h, RDS_EINVAL, "rds_get_u_gt: NULL out");
    if (h->batch > 1) return batch_out(h, out, h->d64 + h->plane + h->origin, 8, 0, on_device);
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(h, cudaMemcpy2DAsync(out, sizeof(double) * h->W, h->d64 + h->plane + h->origin,
                            sizeof(double) * h->pitch, sizeof(double) * h->W, h->H, kind,
                            h->stream));
    if (!on_device) CK(h, cudaStreamSynchronize(h->stream));
    return RDS_OK;
}

int rds_compare_gt(rds_t *h, float eps, double *e1, double *e2) {
    NEED_SOLVED("rds_compare_gt");
    if (!h->have_gt) return fail(h, RDS_ESTATE, "rds_compare_gt: no rds_solve_gt has run yet");
    if (!e1 || !e2) return fail(h, RDS_EINVAL, "rds_compare_gt: NULL out");
    if (!(eps >= 0.0f && eps <= 1.0f))
        return fail(h, RDS_EINVAL, "rds_compare_gt: eps=%g must be in [0, 1]", eps);
    CK(h, launch_compare(h->at(h->u), h->d64 + h->plane + h->origin, h->pitch, (int)h->H,
                         (int)h->W, eps, h->part64, h->cmp_out, h->stream));
    double r[2];
    CK(h, cudaMemcpyAsync(r, h->cmp_out, sizeof r, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    *e1 = r[0];
    *e2 = r[1];
    return RDS_OK;
}

int rds_check_frame(rds_t *h, int64_t *bad_count) {
    if (!h || !bad_count) return fail(h, RDS_EINVAL, "rds_check_frame: NULL argument");
    {
        const int rc = resolve(h);
        if (rc) return rc;
    }
    unsigned long long *bad = nullptr;
    CK(h, cudaMalloc(&bad, sizeof *bad));
    cudaError_t e = cudaMemsetAsync(bad, 0, sizeof *bad, h->stream);
    struct P {
        const void *base;
        int elt, swz;
        double expect;
    };
    const P planes[] = {{h->p1[0], 4, 1, 0.0}, {h->p1[1], 4, 1, 0.0}, {h->p2[0], 4, 1, 0.0},
                        {h->p2[1], 4, 1, 0.0}, {h->v[0], 4, 1, 0.0},  {h->v[1], 4, 1, 0.0},
                        {h->c, 4, 1, INFINITY},  {h->u, 4, 0, 0.0},    {h->f, 4, 0, 0.0},
                        {h->z, 4, 0, 0.0},       {h->mask, 1, 0, 0.0}, {h->lab, 1, 0, 0.0}};
    for (const P &q : planes)
        if (e == cudaSuccess)
            e = launch_frame_check(q.base, q.elt, h->pitch, h->rows_alloc, PAD_R, PAD_C,
                                   (int)h->H, (int)h->W, q.swz, q.expect, bad, h->stream);
    unsigned long long n = 0;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&n, bad, sizeof n, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(bad);
    CK(h, e);
    *bad_count = (int64_t)n;
    return RDS_OK;
}

int rds_kfuse_supported(int32_t *out, int cap) { return kf_list(out, cap); }

const char *rds_last_error(rds_t *h) {
    if (h) return h->err.c_str();
    return g_last_error.c_str();
}

const char *rds_version(void) { return "librds 0.1 (sm_100a)"; }

}  // extern "C"
