// rds3_api.cu -- host side of the 3-D volume path of librds (f4): the rds3_* calls of
// include/rds.h.  A handle owns a padded volume per field (internal.h VOL_*); rds3_solve
// enqueues K1 (k_vol_setup) and K launches of k_vol_step (one iteration each, the last one
// writing u and the mask) on ping-pong buffers, replayed from a cached CUDA graph.
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

struct rds3_handle {
    int64_t D = 0, H = 0, W = 0;
    int64_t pitch = 0, plane = 0, vol = 0, origin = 0;
    float *z = nullptr, *P = nullptr, *f = nullptr, *c = nullptr, *u = nullptr;
    float *p1[2] = {}, *p2[2] = {}, *p3[2] = {}, *v[2] = {};
    uint8_t *lab = nullptr, *mask = nullptr;
    float *stage = nullptr;                 // dense staging for host transfers
    unsigned long long *n_rd = nullptr;
    unsigned *absmax_bits = nullptr;
    cudaStream_t own = nullptr, stream = nullptr;
    cudaEvent_t ev[2] = {};
    cudaGraphExec_t graph = nullptr;
    int gkey_iters = -1, gkey_kz = -1, gkey_kf = -1, gkey_kzt = -1;
    int launches = 0;                       // launches of the cached K-loop (final buffer)
    float gkey_tau = 0, gkey_theta = 0;
    bool have_image = false, have_fitting = false, solved = false;
    float c1 = 0, c2 = 0, gamma = 0;
    int cur = 0, kz = 0, iters = 0, opt_kz = 0;
    int opt_kf = 0, kf = 1, kz_tb = 0;     // iterations per pass (k_vol_tb) and its z-chunk
    std::string err;
    float *at(float *b) const { return b + origin; }
    uint8_t *at(uint8_t *b) const { return b + origin; }
};

static int fail3(rds3_t *h, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (h) h->err = buf;
    return code;
}

#define CK3(h, call)                                                                      \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail3((h), e_ == cudaErrorMemoryAllocation ? RDS_ENOMEM : RDS_ECUDA,   \
                         "%s failed: %s", #call, cudaGetErrorString(e_));                 \
    } while (0)

static void free3(rds3_t *h) {
    float *fl[] = {h->z, h->P, h->f, h->c, h->u, h->p1[0], h->p1[1], h->p2[0], h->p2[1],
                   h->p3[0], h->p3[1], h->v[0], h->v[1], h->stage};
    for (float *p : fl)
        if (p) cudaFree(p);
    void *o[] = {h->lab, h->mask, h->n_rd, h->absmax_bits};
    for (void *p : o)
        if (p) cudaFree(p);
    if (h->graph) cudaGraphExecDestroy(h->graph);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->own) cudaStreamDestroy(h->own);
}

extern "C" {

int rds3_create(int64_t D, int64_t H, int64_t W, rds3_t **out) {
    if (!out) return RDS_EINVAL;
    *out = nullptr;
    if (D < 1 || H < 1 || W < 1 || D * H * W > (int64_t(1) << 31)) return RDS_EINVAL;
    rds3_t *h = new (std::nothrow) rds3_t();
    if (!h) return RDS_ENOMEM;
    h->D = D;
    h->H = H;
    h->W = W;
    h->pitch = (VOL_PX_L + W + VOL_PX_R + 31) / 32 * 32;
    h->plane = h->pitch * (VOL_PY_TOP + H + VOL_PY_BOT);
    h->vol = h->plane * (D + 2 * VOL_PZ);
    h->origin = VOL_PZ * h->plane + VOL_PY_TOP * h->pitch + VOL_PX_L;
    auto bad = [&](cudaError_t e) {
        if (e == cudaSuccess) return false;
        free3(h);
        delete h;
        return true;
    };
    if (bad(cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking))) return RDS_ECUDA;
    h->stream = h->own;
    float **zero_planes[] = {&h->z, &h->f, &h->u, &h->p1[0], &h->p1[1], &h->p2[0], &h->p2[1],
                             &h->p3[0], &h->p3[1], &h->v[0], &h->v[1]};
    for (float **pp : zero_planes) {
        if (bad(cudaMalloc(pp, sizeof(float) * h->vol))) return RDS_ENOMEM;
        if (bad(cudaMemsetAsync(*pp, 0, sizeof(float) * h->vol, h->stream))) return RDS_ECUDA;
    }
    if (bad(cudaMalloc(&h->c, sizeof(float) * h->vol))) return RDS_ENOMEM;
    if (bad(launch_fill_frame(h->c, h->vol, INFINITY, h->stream))) return RDS_ECUDA;
    if (bad(cudaMalloc(&h->lab, h->vol)) || bad(cudaMemsetAsync(h->lab, 0, h->vol, h->stream)))
        return RDS_ENOMEM;
    if (bad(cudaMalloc(&h->mask, h->vol)) || bad(cudaMemsetAsync(h->mask, 0, h->vol, h->stream)))
        return RDS_ENOMEM;
    if (bad(cudaMalloc(&h->stage, sizeof(float) * D * H * W))) return RDS_ENOMEM;
    if (bad(cudaMalloc(&h->n_rd, sizeof(unsigned long long)))) return RDS_ENOMEM;
    if (bad(cudaMalloc(&h->absmax_bits, sizeof(unsigned)))) return RDS_ENOMEM;
    for (auto &e : h->ev)
        if (bad(cudaEventCreate(&e))) return RDS_ECUDA;
    if (bad(cudaStreamSynchronize(h->stream))) return RDS_ECUDA;
    *out = h;
    return RDS_OK;
}

int rds3_destroy(rds3_t *h) {
    if (!h) return RDS_OK;
    if (h->stream) cudaStreamSynchronize(h->stream);
    free3(h);
    delete h;
    return RDS_OK;
}

int rds3_set_stream(rds3_t *h, void *stream) {
    if (!h) return RDS_EINVAL;
    cudaStream_t s = stream ? (cudaStream_t)stream : h->own;
    if (s != h->stream) {
        CK3(h, cudaStreamSynchronize(h->stream));
        h->stream = s;
        if (h->graph) {
            cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
        }
    }
    return RDS_OK;
}

// dense (D, H, W) float32 -> padded volume (through the staging buffer for host input)
static int vol_in(rds3_t *h, float *vol, const float *src, int on_device) {
    const float *dsrc = src;
    if (!on_device) {
        CK3(h, cudaMemcpyAsync(h->stage, src, sizeof(float) * h->D * h->H * h->W,
                               cudaMemcpyHostToDevice, h->stream));
        dsrc = h->stage;
    }
    CK3(h, launch_vol_copy_f32(h->at(vol), dsrc, h->plane, h->pitch, (int)h->D, (int)h->H,
                               (int)h->W, 1, h->stream));
    if (!on_device) CK3(h, cudaStreamSynchronize(h->stream));
    return RDS_OK;
}

int rds3_set_kz(rds3_t *h, int32_t kz) {
    if (!h || kz < 0) return RDS_EINVAL;
    h->opt_kz = kz;
    return RDS_OK;
}

int rds3_set_kfuse(rds3_t *h, int32_t kf) {
    if (!h) return RDS_EINVAL;
    if (kf < 0 || kf > VOL_TB_MAX)
        return fail3(h, RDS_EINVAL, "rds3_set_kfuse: k_fuse=%d not in 0 .. %d", kf, VOL_TB_MAX);
    h->opt_kf = kf;
    return RDS_OK;
}

// 1 if every value of a padded volume (frame included: zeros) is finite
static int vol_finite(rds3_t *h, const float *vol, bool *ok) {
    int *flag = nullptr;
    CK3(h, cudaMalloc(&flag, sizeof(int)));
    int bad = 0;
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), h->stream);
    if (e == cudaSuccess)
        e = launch_check_finite(vol, h->pitch, (int)(h->vol / h->pitch), (int)h->pitch, flag,
                                h->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(flag);
    CK3(h, e);
    *ok = bad == 0;
    return RDS_OK;
}

int rds3_set_image(rds3_t *h, const float *z, int on_device) {
    if (!h || !z) return fail3(h, RDS_EINVAL, "rds3_set_image: NULL argument");
    int rc = vol_in(h, h->z, z, on_device);
    if (rc) return rc;
    bool ok = true;
    if ((rc = vol_finite(h, h->z, &ok))) return rc;
    h->have_image = ok;
    if (!ok) return fail3(h, RDS_EINVAL, "rds3_set_image: non-finite values");
    return RDS_OK;
}

int rds3_set_fitting(rds3_t *h, float c1, float c2, float gamma, const float *P, int on_device) {
    if (!h) return RDS_EINVAL;
    if (!isfinite(c1) || !isfinite(c2) || c1 == c2 || !isfinite(gamma) || gamma < 0.0f ||
        (gamma > 0.0f && !P))
        return fail3(h, RDS_EINVAL, "rds3_set_fitting: need finite c1 != c2, gamma >= 0, P");
    if (gamma > 0.0f) {
        if (!h->P) {
            CK3(h, cudaMalloc(&h->P, sizeof(float) * h->vol));
            CK3(h, cudaMemsetAsync(h->P, 0, sizeof(float) * h->vol, h->stream));
        }
        int rc = vol_in(h, h->P, P, on_device);
        if (rc) return rc;
        bool ok = true;
        if ((rc = vol_finite(h, h->P, &ok))) return rc;
        if (!ok) {
            h->have_fitting = false;
            return fail3(h, RDS_EINVAL, "rds3_set_fitting: P has non-finite values");
        }
    }
    h->c1 = c1;
    h->c2 = c2;
    h->gamma = gamma;
    h->have_fitting = true;
    return RDS_OK;
}

int rds3_fitting_absmax(rds3_t *h, float *out) {
    if (!h || !out) return RDS_EINVAL;
    if (!h->have_image || !h->have_fitting)
        return fail3(h, RDS_ESTATE, "rds3_fitting_absmax: image and fitting must be set");
    CK3(h, cudaMemsetAsync(h->absmax_bits, 0, sizeof(unsigned), h->stream));
    CK3(h, launch_vol_absmax(h->at(h->z), h->gamma != 0.0f ? h->at(h->P) : nullptr, h->plane,
                             h->pitch, (int)h->D, (int)h->H, (int)h->W, h->c1, h->c2, h->gamma,
                             h->absmax_bits, h->stream));
    unsigned bits = 0;
    CK3(h, cudaMemcpyAsync(&bits, h->absmax_bits, sizeof bits, cudaMemcpyDeviceToHost,
                           h->stream));
    CK3(h, cudaStreamSynchronize(h->stream));
    memcpy(out, &bits, sizeof bits);
    return RDS_OK;
}

// The K-loop: kf = 1 one k_vol_step launch per iteration; kf > 1 k_vol_tb launches of kf
// iterations each (the last one of iters mod kf), ping-ponging the state buffers; the last
// launch writes u and the mask.  Returns the launch count in *launches.
static cudaError_t enqueue3(rds3_t *h, int iters, float tau, float theta, int *launches) {
    VolArgs a{};
    a.c = h->at(h->c);
    a.u_out = h->at(h->u);
    a.mask_out = h->at(h->mask);
    a.plane = h->plane;
    a.pitch = h->pitch;
    a.D = (int)h->D;
    a.H = (int)h->H;
    a.W = (int)h->W;
    a.tau = tau;
    a.theta = theta;
    a.inv_theta = 1.0f / theta;
    int cur = h->cur, n = 0;
    for (int it = 0; it < iters;) {
        const int step = h->kf > 1 ? (iters - it < h->kf ? iters - it : h->kf) : 1;
        a.p1_in = h->at(h->p1[cur]);
        a.p2_in = h->at(h->p2[cur]);
        a.p3_in = h->at(h->p3[cur]);
        a.v_in = h->at(h->v[cur]);
        a.p1_out = h->at(h->p1[cur ^ 1]);
        a.p2_out = h->at(h->p2[cur ^ 1]);
        a.p3_out = h->at(h->p3[cur ^ 1]);
        a.v_out = h->at(h->v[cur ^ 1]);
        const bool last = it + step == iters;
        cudaError_t e;
        if (h->kf > 1) {
            a.kz = h->kz_tb;
            e = launch_vol_tb(a, step, last, h->stream);
        } else {
            a.kz = h->kz;
            e = launch_vol_step(a, last, h->stream);
        }
        if (e != cudaSuccess) return e;
        cur ^= 1;
        it += step;
        ++n;
    }
    *launches = n;
    return cudaSuccess;
}

// z-chunk of k_vol_tb<S>: the chunk count whose waves of CTAs (tiles x chunks over the
// resident slots) times the per-CTA plane steps (kz + 3S) is least
static int plan_kz_tb(rds3_t *h, int S) {
    if (h->opt_kz > 0) return (int)(h->opt_kz < h->D ? h->opt_kz : h->D);
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    (void)cudaGetLastError();
    const int64_t tiles = vol_tb_tiles(S, h->H, h->W);
    const int64_t slots = (int64_t)n_sm * vol_tb_blocks_per_sm(S);
    int best_kz = (int)h->D;
    double best = 1e300;
    for (int64_t c = 1; c <= h->D && c <= 512; ++c) {
        const int64_t kz = (h->D + c - 1) / c, ce = (h->D + kz - 1) / kz;
        const int64_t waves = (tiles * ce + slots - 1) / slots;
        const double cost = (double)waves * (double)(kz + 3 * S);
        if (cost < best - 1e-9) {
            best = cost;
            best_kz = (int)kz;
        }
    }
    return best_kz;
}

int rds3_solve(rds3_t *h, float lambda, float theta, float tau, float delta, int32_t iters) {
    if (!h) return RDS_EINVAL;
    if (!(lambda > 0.0f) || !isfinite(lambda) || !(theta > 0.0f) || !isfinite(theta))
        return fail3(h, RDS_EINVAL, "rds3_solve: need finite lambda, theta > 0");
    if (!(tau > 0.0f) || !(tau <= 1.0f / 12.0f))
        return fail3(h, RDS_EINVAL, "rds3_solve: tau=%g must be in (0, 1/12] in 3-D", tau);
    if (isnan(delta) || delta < 0.0f || iters < 0)
        return fail3(h, RDS_EINVAL, "rds3_solve: need delta >= 0, iters >= 0");
    if (!h->have_image || !h->have_fitting)
        return fail3(h, RDS_ESTATE, "rds3_solve: image and fitting must be set first");
    nvtxRangePushA("rds3_solve");
    struct Pop {
        ~Pop() { nvtxRangePop(); }
    } pop;
    // z-chunk per CTA: enough CTAs for ~4 waves of 4 resident CTAs per SM, >= 8 planes
    {
        const int64_t tiles = vol_tiles(h->H, h->W);
        int64_t chunks = (148 * 16 + tiles - 1) / tiles;
        int kz = h->opt_kz > 0 ? h->opt_kz : (int)((h->D + chunks - 1) / chunks);
        if (kz < 8 && h->opt_kz <= 0) kz = 8;
        if (kz > h->D) kz = (int)h->D;
        h->kz = kz;
        h->kf = h->opt_kf > 0 ? h->opt_kf : VOL_TB_DEFAULT;
        h->kz_tb = h->kf > 1 ? plan_kz_tb(h, h->kf) : 0;
    }
    CK3(h, cudaEventRecord(h->ev[0], h->stream));
    VolSetupArgs s{};
    s.z = h->at(h->z);
    s.P = h->gamma != 0.0f ? h->at(h->P) : nullptr;
    s.f = h->at(h->f);
    s.c = h->at(h->c);
    s.u = h->at(h->u);
    s.v0 = h->at(h->v[0]);
    s.v1 = h->at(h->v[1]);
    s.p10 = h->at(h->p1[0]);
    s.p11 = h->at(h->p1[1]);
    s.p20 = h->at(h->p2[0]);
    s.p21 = h->at(h->p2[1]);
    s.p30 = h->at(h->p3[0]);
    s.p31 = h->at(h->p3[1]);
    s.lab = h->at(h->lab);
    s.mask = h->at(h->mask);
    s.n_rd = h->n_rd;
    s.plane = h->plane;
    s.pitch = h->pitch;
    s.D = (int)h->D;
    s.H = (int)h->H;
    s.W = (int)h->W;
    s.c1 = h->c1;
    s.c2 = h->c2;
    s.gamma = h->gamma;
    s.delta = delta;
    s.theta_lambda = theta * lambda;
    CK3(h, cudaMemsetAsync(h->n_rd, 0, sizeof(unsigned long long), h->stream));
    CK3(h, launch_vol_setup(s, h->stream));
    h->cur = 0;
    if (iters > 0) {
        const bool same = h->graph && h->gkey_iters == iters && h->gkey_kz == h->kz &&
                          h->gkey_kf == h->kf && h->gkey_kzt == h->kz_tb &&
                          h->gkey_tau == tau && h->gkey_theta == theta;
        if (!same) {
            if (h->graph) cudaGraphExecDestroy(h->graph);
            h->graph = nullptr;
            cudaStream_t cap;
            CK3(h, cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            cudaGraph_t g = nullptr;
            cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
                cudaStream_t keep = h->stream;
                h->stream = cap;
                const cudaError_t e2 = enqueue3(h, iters, tau, theta, &h->launches);
                h->stream = keep;
                e = cudaStreamEndCapture(cap, &g);
                if (e == cudaSuccess) e = e2;
            }
            if (e == cudaSuccess) e = cudaGraphInstantiate(&h->graph, g, 0);
            if (g) cudaGraphDestroy(g);
            cudaStreamDestroy(cap);
            if (e != cudaSuccess) {
                h->graph = nullptr;
                return fail3(h, RDS_ECUDA, "rds3_solve: graph: %s", cudaGetErrorString(e));
            }
            h->gkey_iters = iters;
            h->gkey_kz = h->kz;
            h->gkey_kf = h->kf;
            h->gkey_kzt = h->kz_tb;
            h->gkey_tau = tau;
            h->gkey_theta = theta;
        }
        CK3(h, cudaGraphLaunch(h->graph, h->stream));
        if (h->launches & 1) h->cur = 1;
    }
    CK3(h, cudaEventRecord(h->ev[1], h->stream));
    h->iters = iters;
    h->solved = true;
    return RDS_OK;
}

static int vol_out_f32(rds3_t *h, float *dst, const float *vol, int on_device) {
    if (!h->solved) return fail3(h, RDS_ESTATE, "rds3: no solve has run yet");
    if (!dst) return fail3(h, RDS_EINVAL, "rds3: NULL out");
    float *d = on_device ? dst : h->stage;
    CK3(h, launch_vol_copy_f32(d, vol + h->origin, h->plane, h->pitch, (int)h->D, (int)h->H,
                               (int)h->W, 0, h->stream));
    if (!on_device) {
        CK3(h, cudaMemcpyAsync(dst, h->stage, sizeof(float) * h->D * h->H * h->W,
                               cudaMemcpyDeviceToHost, h->stream));
        CK3(h, cudaStreamSynchronize(h->stream));
    }
    return RDS_OK;
}

static int vol_out_u8(rds3_t *h, uint8_t *dst, const uint8_t *vol, int on_device) {
    if (!h->solved) return fail3(h, RDS_ESTATE, "rds3: no solve has run yet");
    if (!dst) return fail3(h, RDS_EINVAL, "rds3: NULL out");
    uint8_t *d = on_device ? dst : reinterpret_cast<uint8_t *>(h->stage);
    CK3(h, launch_vol_copy_u8(d, vol + h->origin, h->plane, h->pitch, (int)h->D, (int)h->H,
                              (int)h->W, 0, h->stream));
    if (!on_device) {
        CK3(h, cudaMemcpyAsync(dst, d, (size_t)(h->D * h->H * h->W), cudaMemcpyDeviceToHost,
                               h->stream));
        CK3(h, cudaStreamSynchronize(h->stream));
    }
    return RDS_OK;
}

int rds3_get_u(rds3_t *h, float *out, int on_device) {
    if (!h) return RDS_EINVAL;
    return vol_out_f32(h, out, h->u, on_device);
}
int rds3_get_v(rds3_t *h, float *out, int on_device) {
    if (!h) return RDS_EINVAL;
    return vol_out_f32(h, out, h->v[h->cur], on_device);
}
int rds3_get_p(rds3_t *h, float *rho1, float *rho2, float *rho3, int on_device) {
    if (!h) return RDS_EINVAL;
    int rc = vol_out_f32(h, rho1, h->p1[h->cur], on_device);
    if (!rc) rc = vol_out_f32(h, rho2, h->p2[h->cur], on_device);
    if (!rc) rc = vol_out_f32(h, rho3, h->p3[h->cur], on_device);
    return rc;
}
int rds3_get_mask(rds3_t *h, uint8_t *out, int on_device) {
    if (!h) return RDS_EINVAL;
    return vol_out_u8(h, out, h->mask, on_device);
}
int rds3_get_labels(rds3_t *h, uint8_t *out, int on_device) {
    if (!h) return RDS_EINVAL;
    return vol_out_u8(h, out, h->lab, on_device);
}

int rds3_get_stats(rds3_t *h, int64_t *n_rd, int32_t *iters, int32_t *kz, float *loop_ms) {
    if (!h) return RDS_EINVAL;
    if (!h->solved) return fail3(h, RDS_ESTATE, "rds3_get_stats: no solve has run yet");
    unsigned long long nrd = 0;
    CK3(h, cudaMemcpyAsync(&nrd, h->n_rd, sizeof nrd, cudaMemcpyDeviceToHost, h->stream));
    CK3(h, cudaStreamSynchronize(h->stream));
    if (n_rd) *n_rd = (int64_t)nrd;
    if (iters) *iters = h->iters;
    if (kz) *kz = h->kf > 1 ? h->kz_tb : h->kz;
    if (loop_ms) CK3(h, cudaEventElapsedTime(loop_ms, h->ev[0], h->ev[1]));
    return RDS_OK;
}

const char *rds3_last_error(rds3_t *h) { return h ? h->err.c_str() : ""; }

}  // extern "C"
