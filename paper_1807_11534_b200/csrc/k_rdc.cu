// k_rdc.cu -- f3: the compacted restricted-domain iteration (RDS_OPT_COMPACT).
//
// The paper iterates "only on the restricted domain" (Eq. 7-9).  The dense
// stencil (K3) does that per work item, which cannot skip anything when the band is
// scattered noise (C3: every 8-row band of every strip holds RD pixels).  Here
// the state of the RD pixels alone is stored in compact arrays, in row-major RD order, with
// each pixel's six stencil neighbours as compact indices (or the pinned class of a
// non-RD neighbour: rho = 0 there and v = u0 = 0 / 1).  At low band fractions the whole
// working set (~52 B per RD pixel) stays in L2 and the cost of an iteration scales with the
// number of RD pixels, not with the tiles they touch.
//
// One persistent cooperative kernel runs the K iterations; a grid barrier separates them.
// Pass k (0 <= k <= K) at RD pixel x, with p = rho (reading R-C5/R-C6):
//   k >= 1: u^k(y) = v^{k-1}(y) - theta div p^k(y), v^k(y) = clamp(u^k(y) - theta lambda f(y))
//           for y = x, x+e1, x+e2 (the two neighbours recomputed, so one barrier per pass)
//   k <  K: w^k(y) = div p^k(y) - v^k(y)/theta for the same y, g = grad w^k at x,
//           p^{k+1}(x) = (p^k(x) + tau g) / (1 + tau |g|)
// Every float operation is the dense kernel's, in the same order and rounding (explicit _rn
// intrinsics, the same MUFU sqrt/rcp, c' = 2^-100 theta lambda f with the |c'| and FFMA.SAT
// folds), so the two paths agree value for value (tests/test_gpu_compact.py); the final state
// is scattered back into the dense planes, after which every getter, rds_energy and
// rds_solve_continue work unchanged.
#include <math.h>
#include <stdlib.h>

#include "internal.h"

namespace rds {

namespace {

__device__ __forceinline__ float sqrt_ax(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ax(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// one warp per row: RD pixels per row (labels: 0 Bg, 1 Fg, 2 RD)
__global__ void k_rdc_rowcount(const uint8_t *lab, int64_t pitch, int H, int W, int32_t *cnt) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= H) return;
    const uint8_t *row = lab + (int64_t)i * pitch;
    int c = 0;
    for (int j0 = 0; j0 < W; j0 += 32) {
        const int j = j0 + lane;
        c += __popc(__ballot_sync(0xffffffffu, j < W && row[j] == 2));
    }
    if (lane == 0) cnt[i] = c;
}

// exclusive scan of the row counts (one CTA, fixed order) and the total
__global__ void __launch_bounds__(1024) k_rdc_scan(const int32_t *cnt, int H, int32_t *off,
                                                   int32_t *total) {
    __shared__ int32_t wsum[32];
    __shared__ int32_t carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int b = 0; b < H; b += 1024) {
        const int i = b + tid;
        const int x = i < H ? cnt[i] : 0;
        int incl = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int s = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;  // inclusive over warps
        }
        __syncthreads();
        const int before = carry + (wid > 0 ? wsum[wid - 1] : 0);
        if (i < H) off[i] = before + incl - x;
        __syncthreads();
        if (tid == 0) carry += wsum[31];
        __syncthreads();
    }
    if (tid == 0) *total = carry;
}

// one warp per row: RD pixels get their compact index (row-major order) and a list entry;
// every other pixel its pinned class in the index map
__global__ void k_rdc_fill(const uint8_t *lab, int64_t pitch, int H, int W, const int32_t *off,
                           int32_t *idxmap, int32_t *list) {
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= H) return;
    const uint8_t *row = lab + (int64_t)i * pitch;
    int run = off[i];
    for (int j0 = 0; j0 < W; j0 += 32) {
        const int j = j0 + lane;
        const int l = j < W ? row[j] : 0;
        const unsigned b = __ballot_sync(0xffffffffu, l == 2);
        if (j < W) {
            const int64_t pix = (int64_t)i * W + j;
            if (l == 2) {
                const int r = run + __popc(b & ((1u << lane) - 1u));
                idxmap[pix] = r;
                list[r] = (int32_t)pix;
            } else {
                idxmap[pix] = l == 1 ? RDC_FG : RDC_BG;
            }
        }
        run += __popc(b);
    }
}

// per RD pixel: neighbour codes and the record (rho1, rho2, v, c') from the dense planes
__global__ void k_rdc_gather(const RdcSetup a) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int64_t pix = a.list[r];
        const int i = (int)(pix / a.W), j = (int)(pix - (int64_t)i * a.W);
        const bool top = i == 0, bottom = i == a.H - 1, left = j == 0;
        const bool right = j % a.img_w == a.img_w - 1;  // grad_2 = 0 (per image of a batch)
        // index-map codes of the six neighbours (frame: pinned 0 / Neumann edge)
        const int up = top ? RDC_BG : a.idxmap[pix - a.W];
        const int dn = bottom ? RDC_EDGE : a.idxmap[pix + a.W];
        const int lf = left ? RDC_BG : a.idxmap[pix - 1];
        const int rt = right ? RDC_EDGE : a.idxmap[pix + 1];
        const int dl = (bottom || left) ? RDC_BG : a.idxmap[pix + a.W - 1];
        const int ur = (top || j == a.W - 1) ? RDC_BG : a.idxmap[pix - a.W + 1];
        // packed (see RdcCode): anchors = the RD index of up (else ur) and of down (else dl)
        const unsigned ia = up >= 0 ? up : (ur >= 0 ? ur : 0);
        const unsigned ib = dn >= 0 ? dn : (dl >= 0 ? dl : 0);
        const unsigned fa = rdc_cls(up) | (rdc_cls(ur) << 2) | (rdc_cls(lf) << 4);
        const unsigned fb = rdc_cls(dn) | (rdc_cls(dl) << 2) | (rdc_cls(rt) << 4);
        a.code[r] = make_uint2(ia | (fa << RDC_IDX_BITS), ib | (fb << RDC_IDX_BITS));
        const int64_t o = (int64_t)i * a.pitch + swz(j);
        a.rec[r] = make_float4(a.p1plane[o], a.p2plane[o], a.vplane[o], a.cplane[o]);
        a.u[r] = a.uplane[(int64_t)i * a.pitch + j];  // u^0 = u0 (a check after iteration 1)
    }
}

// final state back into the dense planes (rho, v swizzled; u, mask natural order).  After l
// iterations rho^l is in the buffer pass l read (rec[l & 1]) and v^l in the one it wrote.
__global__ void k_rdc_scatter(const RdcSetup a, const float4 *rec0, const float4 *rec1, int K,
                              const StopRecord *stop) {
    const int l = stop ? stop->iters : K;
    const float4 *Pb = (l & 1) ? rec1 : rec0, *Vb = (l & 1) ? rec0 : rec1;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int64_t pix = a.list[r];
        const int i = (int)(pix / a.W), j = (int)(pix - (int64_t)i * a.W);
        const int64_t o = (int64_t)i * a.pitch + swz(j), on = (int64_t)i * a.pitch + j;
        const float4 x = Pb[r];
        a.p1plane[o] = x.x;
        a.p2plane[o] = x.y;
        a.vplane[o] = Vb[r].z;
        const float u = a.u[r];
        a.uplane[on] = u;
        a.mask[on] = u > 0.5f;
    }
}

// Record loads: RDC_L1 = 1 caches them in L1 (each record is read by up to 7 pixels of a pass;
// the acquire load that ends every grid barrier invalidates the SM's L1, so no line from an
// earlier pass survives), 0 reads through L2 only (ld.global.cg).
#ifndef RDC_L1
#define RDC_L1 1
#endif
__device__ __forceinline__ float4 ld_rec(const float4 *p) {
#if RDC_L1
    return *p;
#else
    return __ldcg(p);
#endif
}

// the record of a neighbour code: an RD pixel's (rho1, rho2, v, c') from this pass's buffer
// (rewritten by other CTAs before the last barrier), or a pinned pixel's (0, 0, u0, -):
// rho = 0 on Fg u Bg (Eq. 8), v = u0
__device__ __forceinline__ float4 rec_at(const float4 *B, int code) {
    if (code >= 0) return ld_rec(B + code);
    return make_float4(0.0f, 0.0f, code == RDC_FG ? 1.0f : 0.0f, 0.0f);
}

// Grid-wide barrier number k (1, 2, ...): one release-add per CTA on a monotone counter,
// then an acquire spin until all gridDim.x CTAs have arrived k times.  (A two-level version
// with group counters measured slower: its serial fence/atomic chain outweighs the
// contention of ~300 arrivals on one address.)
__device__ __forceinline__ void grid_barrier(unsigned long long *bar, unsigned long long k) {
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

}  // namespace

// A pixel's neighbour codes (constant over the solve), decoded from its packed pair.
struct PixConst {
    int r, up, dn, lf, rt, dl, ur;
};

__device__ __forceinline__ int cls_code(unsigned c) {  // pinned class -> neighbour code
    return c == RDC_C_FG ? RDC_FG : (c == RDC_C_EDGE ? RDC_EDGE : RDC_BG);
}

__device__ __forceinline__ PixConst decode(uint2 w, int r) {
    const int ia = (int)(w.x & RDC_IDX_MASK), ib = (int)(w.y & RDC_IDX_MASK);
    const unsigned fa = w.x >> RDC_IDX_BITS, fb = w.y >> RDC_IDX_BITS;
    const unsigned cu = fa & 3, cur = (fa >> 2) & 3, cl = fa >> 4;
    const unsigned cd = fb & 3, cdl = (fb >> 2) & 3, cr = fb >> 4;
    PixConst q;
    q.r = r;
    // row-major RD order: (i, j +- 1) are r +- 1; (i-1, j+1) follows (i-1, j), (i+1, j-1)
    // precedes (i+1, j) when both are RD
    q.up = cu == RDC_C_RD ? ia : cls_code(cu);
    q.ur = cur == RDC_C_RD ? (cu == RDC_C_RD ? ia + 1 : ia) : cls_code(cur);
    q.dn = cd == RDC_C_RD ? ib : cls_code(cd);
    q.dl = cdl == RDC_C_RD ? (cd == RDC_C_RD ? ib - 1 : ib) : cls_code(cdl);
    q.lf = cl == RDC_C_RD ? r - 1 : cls_code(cl);
    q.rt = cr == RDC_C_RD ? r + 1 : cls_code(cr);
    return q;
}

// v^k of a neighbour y (code, record, div p^k there) from v^{k-1}: Eq. 7 and 9; pass 0: v^0
__device__ __forceinline__ float v_of(int code, const float4 &y, float dy, int k, float theta) {
    if (code < 0 || k == 0) return y.z;  // pinned u0 / v^0
    return __saturatef(__fmaf_rn(y.w, -0x1p100f, __fmaf_rn(dy, -theta, y.z)));
}

// Pass k at one RD pixel (see the header comment): from its record X = (rho^k, v^{k-1}, c')
// and its neighbours' records in B, the new record (rho^{k+1}, v^k, c') -- the same float
// operations as K3 -- and u^k (ux).  A decoupled pixel (no RD neighbour, k_rdc_iso) never
// dereferences B: every neighbour is a pinned constant.
__device__ __forceinline__ float4 pix_next(const PixConst &q, const float4 &X, const float4 *B,
                                           int k, int K, float tau, float theta,
                                           float inv_theta, float &ux) {
    const float4 Up = rec_at(B, q.up), Lf = rec_at(B, q.lf);
    // div p^k = (p1 - p1(x - e1)) + (p2 - p2(x - e2))
    const float dx = __fadd_rn(__fsub_rn(X.x, Up.x), __fsub_rn(X.y, Lf.y));
    ux = __fmaf_rn(dx, -theta, X.z);
    const float vx = k == 0 ? X.z : __saturatef(__fmaf_rn(X.w, -0x1p100f, ux));
    if (k == K) return make_float4(X.x, X.y, vx, X.w);  // last pass: u^K and v^K only
    const float wx = __fmaf_rn(vx, -inv_theta, dx);
    float g1 = 0.0f, g2 = 0.0f;
    if (q.dn != RDC_EDGE) {  // grad_1 = 0 on row H-1
        const float4 D = rec_at(B, q.dn), DL = rec_at(B, q.dl);
        const float dd = __fadd_rn(__fsub_rn(D.x, X.x), __fsub_rn(D.y, DL.y));
        g1 = __fsub_rn(__fmaf_rn(v_of(q.dn, D, dd, k, theta), -inv_theta, dd), wx);
    }
    if (q.rt != RDC_EDGE) {  // grad_2 = 0 on an image's last column
        const float4 R = rec_at(B, q.rt), UR = rec_at(B, q.ur);
        const float dr = __fadd_rn(__fsub_rn(R.x, UR.x), __fsub_rn(R.y, X.y));
        g2 = __fsub_rn(__fmaf_rn(v_of(q.rt, R, dr, k, theta), -inv_theta, dr), wx);
    }
    const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(X.w)));
    const float rr = rcp_ax(__fmaf_rn(sqrt_ax(s), tau, 1.0f));
    return make_float4(__fmul_rn(__fmaf_rn(g1, tau, X.x), rr),
                       __fmul_rn(__fmaf_rn(g2, tau, X.y), rr), vx, X.w);
}

// Pass k at one RD pixel, reading records (rho^k, v^{k-1}, c') from B and writing
// (rho^{k+1}, v^k, c') to O.
__device__ __forceinline__ void pix_pass(const PixConst &q, const float4 *B, float4 *O,
                                         float *U, int k, int K, float tau, float theta,
                                         float inv_theta, bool chk, bool wr_u, float &su,
                                         float &sv) {
    const float4 X = ld_rec(B + q.r);
    float ux;
    const float4 Y = pix_next(q, X, B, k, K, tau, theta, inv_theta, ux);
    if (chk) {  // the stopping sums of iteration k: u^k - u^{k-1}, v^k - v^{k-1}
        const float du = ux - U[q.r], dv = Y.z - X.z;
        su += du * du;
        sv += dv * dv;
    }
    if (wr_u) U[q.r] = ux;  // an RD pixel reports u itself (u0 only off RD)
    O[q.r] = Y;
}

// Decoupled RD pixels (the split, RDS_RDC_SPLIT; fixed-K solves).  The six stencil neighbours
// come in symmetric pairs (up/down, left/right, up-right/down-left), so a pixel none of whose
// six neighbours is RD reads no other record and no other pixel reads its record: its K
// iterations depend on its own state and pinned constants alone (Eq. 7-9 with rho = 0 and
// v = u0 off RD).  At the scattered noise bands of C3 (RD density p ~ 0.1) that is about
// (1 - p)^6 ~ half of all RD pixels.  They run as one independent thread each, the record in
// registers for all K passes, no grid barrier; the grid-barrier kernel iterates the coupled
// rest through an index list.  Same float operations, so the result is the same bits.
// The one asymmetric pair is an image seam of a batch: the last column's right neighbour is
// EDGE (grad_2 = 0) while the next image's first column still reads it as its left one, so a
// right neighbour of class EDGE counts as coupled (also on the last column of the frame:
// a few pixels more on the barrier path, never a wrong split).
__device__ __forceinline__ bool rdc_coupled(uint2 w) {
    const unsigned fa = w.x >> RDC_IDX_BITS, fb = w.y >> RDC_IDX_BITS;
    const unsigned f = fa | (fb << 6);  // classes: up, ur, lf, dn, dl, rt (2 bits each)
    bool any = (f >> 10) == RDC_C_EDGE;
#pragma unroll
    for (int e = 0; e < 6; ++e) any |= ((f >> (2 * e)) & 3u) == RDC_C_RD;
    return any;
}

namespace {

constexpr int SPLIT_CHUNK = 1024;  // records per CTA of the split (one per thread)

__global__ void __launch_bounds__(SPLIT_CHUNK) k_rdc_split_count(const uint2 *code, int n,
                                                                  int32_t *cnt) {
    const int r = blockIdx.x * SPLIT_CHUNK + threadIdx.x;
    const int c = __syncthreads_count(r < n && rdc_coupled(__ldg(code + r)));
    if (threadIdx.x == 0) cnt[blockIdx.x] = c;
}

// coupled records in ascending order into cpl[off[b] ...], decoupled ones into
// iso[b * SPLIT_CHUNK - off[b] ...] (also ascending)
__global__ void __launch_bounds__(SPLIT_CHUNK) k_rdc_split_fill(const uint2 *code, int n,
                                                                 const int32_t *off,
                                                                 int32_t *cpl, int32_t *iso) {
    __shared__ int wc[SPLIT_CHUNK / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int r = blockIdx.x * SPLIT_CHUNK + t;
    const bool in = r < n;
    const bool c = in && rdc_coupled(__ldg(code + r));
    const unsigned b = __ballot_sync(0xffffffffu, c);
    if (lane == 0) wc[w] = __popc(b);
    __syncthreads();
    int before = 0;  // coupled records of the earlier warps of this chunk
    for (int i = 0; i < w; ++i) before += wc[i];
    const int pc = before + __popc(b & ((1u << lane) - 1u));  // coupled before r in the chunk
    if (!in) return;
    if (c)
        cpl[off[blockIdx.x] + pc] = r;
    else
        iso[blockIdx.x * SPLIT_CHUNK - off[blockIdx.x] + (t - pc)] = r;
}

__global__ void __launch_bounds__(256) k_rdc_iso(const RdcIter a, const int32_t *iso, int n_iso) {
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_iso; i += gridDim.x * blockDim.x) {
        const int r = iso[i];
        const PixConst q = decode(__ldg(a.code + r), r);
        float4 X = a.rec[0][r];  // the gathered start state (pass 0 reads rec[0])
        float ux = 0.0f;
        for (int k = 0; k <= a.K; ++k) X = pix_next(q, X, nullptr, k, a.K, tau, theta, inv_theta, ux);
        // as the barrier kernel leaves it: rho^K in the buffer pass K read, v^K in the one it
        // wrote (k_rdc_scatter), u^K in u (written from pass 1 on)
        a.rec[0][r] = X;
        a.rec[1][r] = X;
        if (a.K >= 1) a.u[r] = ux;
    }
}


// ---------------------------------------------------------------------------------------
// Grouped coupled pixels (RDS_OPT_RDC_SPLIT = 2; fixed-K solves).  The coupled records form a
// graph (an edge wherever one record reads another); at the scattered noise bands the compact
// path serves (RD density well under the site-percolation threshold of the six-neighbour
// lattice) its connected components are small.  A component read by no record outside it and
// reading none can run all K passes inside ONE warp or CTA, its records exchanged through
// shared memory with a warp / CTA barrier per pass -- no grid barrier, no L2 round trip.
// Same float operations (pix_next), so the same bits whichever kernel owns a pixel.
//
// Setup: rounds of min-label propagation over the coupled list (pull and push along every
// read edge, one pointer jump) until a round lowers no label (at most GRP_ROUNDS_MAX), then
// every record checks that all its neighbours carry its
// label ("settled"); a label all of whose records are settled is exactly one component (it is
// closed under adjacency and every member reached the label's own record).  Components of up
// to 1024 settled records get power-of-two slot ranges (classes 2 .. 1024) in a slot array
// ordered by falling class inside three segments (warp: <= 32, CTA of 256, CTA of 1024), so
// no range straddles its block; everything else (unsettled after the last round, or larger) stays on
// the grid-barrier kernel through the fallback list.  Slot order within a class comes from
// atomic counters: it varies from run to run, the values do not.
// ---------------------------------------------------------------------------------------
constexpr int GRP_BATCH = 4, GRP_ROUNDS_MAX = 16;
constexpr bool GRP_2PH_DEFAULT = false;  // two-phase passes (grp_body2); RDS_GRP_2PH overrides

template <typename F>
__device__ __forceinline__ void for_rd_nbrs(const PixConst &q, F f) {
    if (q.up >= 0) f(q.up);
    if (q.ur >= 0) f(q.ur);
    if (q.lf >= 0) f(q.lf);
    if (q.dn >= 0) f(q.dn);
    if (q.dl >= 0) f(q.dl);
    if (q.rt >= 0) f(q.rt);
}

__global__ void k_grp_init(const int32_t *cpl, int nc, int32_t *lab, int32_t *cnt, int32_t *bad,
                           int32_t *cidx) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
        const int r = cpl[i];
        lab[r] = r;
        cnt[r] = 0;
        bad[r] = 0;
        cidx[r] = -1;  // fallback unless k_grp_class finds a settled component rooted here
    }
}

// one round: labels only fall and always name a record of the same component; *changed is
// raised when any label fell (a round that lowers nothing is a fixed point: every edge joins
// equal labels, so every component carries one label)
__global__ void k_grp_prop(const uint2 *code, const int32_t *cpl, int nc, int32_t *lab,
                           int32_t *changed) {
    bool any = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
        const int r = cpl[i];
        const PixConst q = decode(__ldg(code + r), r);
        volatile int32_t *L = lab;
        int m = L[r];
        for_rd_nbrs(q, [&](int nb) { m = min(m, (int)L[nb]); });
        m = min(m, (int)L[m]);
        if (m < L[r]) {
            atomicMin(lab + r, m);
            any = true;
        }
        for_rd_nbrs(q, [&](int nb) {
            if (m < L[nb]) {
                atomicMin(lab + nb, m);
                any = true;
            }
        });
    }
    if (any) *changed = 1;
}

__global__ void k_grp_count(const uint2 *code, const int32_t *cpl, int nc, const int32_t *lab,
                            int32_t *cnt, int32_t *bad, int32_t *rank) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nc; i += gridDim.x * blockDim.x) {
        const int r = cpl[i];
        const PixConst q = decode(__ldg(code + r), r);
        const int l = lab[r];
        for_rd_nbrs(q, [&](int nb) {
            const int ln = lab[nb];
            if (ln != l) {  // an edge between two labels spoils both
                bad[l] = 1;
                bad[ln] = 1;
            }
        });
        rank[r] = atomicAdd(cnt + l, 1);
    }
}

// roots: class k (slot range 2^k, k = 1 .. 10) and the component's index within its class,
// packed as k << 26 | index; -1 (k_grp_init) = fallback: a spoiled or oversized label, or one
// whose own record moved on to a smaller label.  ctr[k] = components of class k, ctr[11] =
// grouped records.
__global__ void __launch_bounds__(256)
k_grp_class(const int32_t *cpl, int nc, const int32_t *lab, const int32_t *cnt,
            const int32_t *bad, int32_t *cidx, int32_t *ctr) {
    // one record per thread; the class counters go through shared memory, one global atomic
    // per class and CTA (300 K roots on eleven addresses cost 190 us at C3 delta = .1)
    __shared__ int32_t sc[12], sb[12];
    if (threadIdx.x < 12) sc[threadIdx.x] = 0;
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int r = -1, k = 0, loc = 0;
    if (i < nc) {
        r = cpl[i];
        const int s = lab[r] == r ? cnt[r] : 0;
        if (s > 0 && !bad[r] && s <= 1024) {
            k = 1;
            while ((1 << k) < s) ++k;
            loc = atomicAdd(sc + k, 1);
            atomicAdd(sc + 11, s);
        }
    }
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x < 12 && sc[threadIdx.x] > 0)
        sb[threadIdx.x] = atomicAdd(ctr + threadIdx.x, sc[threadIdx.x]);
    __syncthreads();
    if (k > 0) cidx[r] = (k << 26) | (sb[k] + loc);
}

struct GrpBases {
    int base[11];  // first slot of class k
};

__global__ void k_grp_fill(const int32_t *cpl, int nc, const int32_t *lab, const int32_t *cidx,
                           const int32_t *rank, const GrpBases gb, int32_t *slots, int32_t *lpos,
                           int32_t *fb, int32_t *nfb) {
    const int n32 = (nc + 31) & ~31;  // whole warps: the ballot below needs every lane
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += gridDim.x * blockDim.x) {
        const bool in = i < nc;
        const int r = in ? cpl[i] : 0;
        const int ci = in ? cidx[lab[r]] : 0;
        const bool f = in && ci < 0;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        const int lane = threadIdx.x & 31;
        int p0 = 0;
        if (b && lane == 0) p0 = atomicAdd(nfb, __popc(b));
        p0 = __shfl_sync(0xffffffffu, p0, 0);
        if (f) fb[p0 + __popc(b & ((1u << lane) - 1u))] = r;
        if (in && ci >= 0) {
            const int k = ci >> 26, idx = ci & ((1 << 26) - 1);
            const int pos = gb.base[k] + (idx << k) + rank[r];
            slots[pos] = r;
            lpos[r] = pos & (k <= 5 ? 31 : k <= 8 ? 255 : 1023);
        }
    }
}

// K passes of the grouped records: block of T slots (T = 32: a warp of a 256-thread CTA),
// records in registers, exchanged through two alternating shared-memory rows.  Passes
// 1 .. K-1 run without class tests in the arithmetic (see the presets below); a missing
// forward neighbour (EDGE) is a select on the difference.  Same operations in the same order
// as pix_next.
template <int T>
__device__ __forceinline__ void grp_body(const RdcIter &a, const int32_t *slots,
                                         const int32_t *lpos, int first, int nslots, int blk,
                                         float4 (*sm)[T == 32 ? 256 : T]) {
    constexpr int NT = T == 32 ? 256 : T;
    const int i = blk * NT + threadIdx.x;
    const int r = i < nslots ? slots[first + i] : -1;
    const bool act = r >= 0;
    const int own = threadIdx.x;
    const int blk0 = T == 32 ? (threadIdx.x & ~31) : 0;  // first slot of this block in sm rows
    PixConst q{};
    float4 X = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    // passes 1 .. K-1: what the pass reads of each neighbour, preset to the pinned record
    // (rho = 0, v = u0, c' = +inf on Bg / the frame, -inf on Fg: the FFMA.SAT of the v-step
    // then returns u0, as K3's c' fold does) and reloaded every pass only where the neighbour
    // is RD -- a lane's neighbour classes never change, so pinned ones cost no shared load
    int iu = -1, iur = -1, il = -1, id = -1, idl = -1, ir = -1;  // shared-row indices (RD only)
    float upx = 0.0f, lfy = 0.0f, dly = 0.0f, urx = 0.0f;
    float4 D = make_float4(0.0f, 0.0f, 0.0f, INFINITY), R = D;
    bool e1 = false, e2 = false;
    if (act) {
        q = decode(__ldg(a.code + r), r);
        auto loc = [&](int c) { return c >= 0 ? blk0 + lpos[c] : c; };
        q.up = loc(q.up);
        q.ur = loc(q.ur);
        q.lf = loc(q.lf);
        q.dn = loc(q.dn);
        q.dl = loc(q.dl);
        q.rt = loc(q.rt);
        iu = q.up;
        iur = q.ur;
        il = q.lf;
        id = q.dn;
        idl = q.dl;
        ir = q.rt;
        if (q.dn == RDC_FG) D = make_float4(0.0f, 0.0f, 1.0f, -INFINITY);
        if (q.rt == RDC_FG) R = make_float4(0.0f, 0.0f, 1.0f, -INFINITY);
        e1 = q.dn == RDC_EDGE;
        e2 = q.rt == RDC_EDGE;
        X = a.rec[0][r];
    }
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    const int K = a.K;
    float ux = 0.0f;
    auto pass = [&](const int k, float4 *B) {
        if (act) B[own] = X;
        if (T == 32)
            __syncwarp();
        else
            __syncthreads();
        if (!act) return;
        if (k == 0 || k == K) {
            X = pix_next(q, X, B, k, K, tau, theta, inv_theta, ux);
            return;
        }
        if (iu >= 0) upx = B[iu].x;
        if (il >= 0) lfy = B[il].y;
        if (id >= 0) D = B[id];
        if (idl >= 0) dly = B[idl].y;
        if (ir >= 0) R = B[ir];
        if (iur >= 0) urx = B[iur].x;
        const float dx = __fadd_rn(__fsub_rn(X.x, upx), __fsub_rn(X.y, lfy));
        ux = __fmaf_rn(dx, -theta, X.z);
        const float vx = __saturatef(__fmaf_rn(X.w, -0x1p100f, ux));
        const float wx = __fmaf_rn(vx, -inv_theta, dx);
        const float dd = __fadd_rn(__fsub_rn(D.x, X.x), __fsub_rn(D.y, dly));
        const float vd = __saturatef(__fmaf_rn(D.w, -0x1p100f, __fmaf_rn(dd, -theta, D.z)));
        float g1 = __fsub_rn(__fmaf_rn(vd, -inv_theta, dd), wx);
        g1 = e1 ? 0.0f : g1;
        const float dr = __fadd_rn(__fsub_rn(R.x, urx), __fsub_rn(R.y, X.y));
        const float vr = __saturatef(__fmaf_rn(R.w, -0x1p100f, __fmaf_rn(dr, -theta, R.z)));
        float g2 = __fsub_rn(__fmaf_rn(vr, -inv_theta, dr), wx);
        g2 = e2 ? 0.0f : g2;
        const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(X.w)));
        const float rr = rcp_ax(__fmaf_rn(sqrt_ax(s), tau, 1.0f));
        X = make_float4(__fmul_rn(__fmaf_rn(g1, tau, X.x), rr),
                        __fmul_rn(__fmaf_rn(g2, tau, X.y), rr), vx, X.w);
    };
    int k = 0;
    for (; k + 1 <= K; k += 2) {
        pass(k, sm[0]);
        pass(k + 1, sm[1]);
    }
    if (k <= K) pass(k, sm[0]);
    if (act) {  // as k_rdc_iso leaves it
        a.rec[0][r] = X;
        a.rec[1][r] = X;
        if (K >= 1) a.u[r] = ux;
    }
}

// Two-phase form of the same passes (RDS_GRP_2PH=1): a pass publishes w = div rho - v / theta
// of every pixel (phase A), then takes grad w from the neighbours' published w (phase B) --
// what K3 does with its stage state -- instead of recomputing the down / right neighbours' w
// from their whole records.  A pinned neighbour's w is formed locally (its rho = 0, v = u0).
// Per pass 3 shared stores and about 4 shared loads of 4 bytes instead of a 16-byte store and
// two 16-byte loads plus four of 4 bytes; two block barriers instead of one.  Same operations
// on the same operands in the same order, so the same bits.
template <int T>
__device__ __forceinline__ void grp_body2(const RdcIter &a, const int32_t *slots,
                                          const int32_t *lpos, int first, int nslots, int blk,
                                          float *sm) {
    constexpr int NT = T == 32 ? 256 : T;
    float *const p1a = sm, *const p2a = sm + NT, *const p1b = sm + 2 * NT, *const p2b = sm + 3 * NT,
                 *const Wp = sm + 4 * NT;
    const int i = blk * NT + threadIdx.x;
    const int r = i < nslots ? slots[first + i] : -1;
    const bool act = r >= 0;
    const int own = threadIdx.x;
    const int blk0 = T == 32 ? (threadIdx.x & ~31) : 0;
    float4 X = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    int iu = -1, iur = -1, il = -1, id = -1, idl = -1, ir = -1;
    float u0d = 0.0f, u0r = 0.0f;
    bool e1 = false, e2 = false;
    if (act) {
        const PixConst q = decode(__ldg(a.code + r), r);
        auto loc = [&](int c) { return c >= 0 ? blk0 + lpos[c] : -1; };
        iu = loc(q.up);
        iur = loc(q.ur);
        il = loc(q.lf);
        id = loc(q.dn);
        idl = loc(q.dl);
        ir = loc(q.rt);
        u0d = q.dn == RDC_FG ? 1.0f : 0.0f;
        u0r = q.rt == RDC_FG ? 1.0f : 0.0f;
        e1 = q.dn == RDC_EDGE;
        e2 = q.rt == RDC_EDGE;
        X = a.rec[0][r];
        p1a[own] = X.x;
        p2a[own] = X.y;
    }
    auto sync = [&]() {
        if (T == 32)
            __syncwarp();
        else
            __syncthreads();
    };
    sync();
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    const int K = a.K;
    float ux = 0.0f;
    auto pass = [&](const int k, const float *p1, const float *p2, float *q1, float *q2) {
        float dx = 0.0f, vx = 0.0f, wx = 0.0f;
        if (act) {
            const float upx = iu >= 0 ? p1[iu] : 0.0f, lfy = il >= 0 ? p2[il] : 0.0f;
            dx = __fadd_rn(__fsub_rn(X.x, upx), __fsub_rn(X.y, lfy));
            ux = __fmaf_rn(dx, -theta, X.z);
            vx = k == 0 ? X.z : __saturatef(__fmaf_rn(X.w, -0x1p100f, ux));
            wx = __fmaf_rn(vx, -inv_theta, dx);
            Wp[own] = wx;
        }
        sync();
        if (act) {
            float wd, wr;
            if (id >= 0) {
                wd = Wp[id];
            } else {
                const float dly = idl >= 0 ? p2[idl] : 0.0f;
                wd = __fmaf_rn(u0d, -inv_theta, __fadd_rn(__fsub_rn(0.0f, X.x), __fsub_rn(0.0f, dly)));
            }
            if (ir >= 0) {
                wr = Wp[ir];
            } else {
                const float urx = iur >= 0 ? p1[iur] : 0.0f;
                wr = __fmaf_rn(u0r, -inv_theta, __fadd_rn(__fsub_rn(0.0f, urx), __fsub_rn(0.0f, X.y)));
            }
            const float g1 = e1 ? 0.0f : __fsub_rn(wd, wx), g2 = e2 ? 0.0f : __fsub_rn(wr, wx);
            const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(X.w)));
            const float rr = rcp_ax(__fmaf_rn(sqrt_ax(s), tau, 1.0f));
            X = make_float4(__fmul_rn(__fmaf_rn(g1, tau, X.x), rr),
                            __fmul_rn(__fmaf_rn(g2, tau, X.y), rr), vx, X.w);
            q1[own] = X.x;
            q2[own] = X.y;
        }
        sync();
    };
    int k = 0;
    for (; k + 2 <= K; k += 2) {
        pass(k, p1a, p2a, p1b, p2b);
        pass(k + 1, p1b, p2b, p1a, p2a);
    }
    if (k + 1 <= K) {
        pass(k, p1a, p2a, p1b, p2b);
        ++k;
    }
    if (act) {  // pass K: u^K and v^K only (rho^K stays); k == K here, rows of parity K
        const float *p1 = (K & 1) ? p1b : p1a, *p2 = (K & 1) ? p2b : p2a;
        const float upx = iu >= 0 ? p1[iu] : 0.0f, lfy = il >= 0 ? p2[il] : 0.0f;
        const float dx = __fadd_rn(__fsub_rn(X.x, upx), __fsub_rn(X.y, lfy));
        ux = __fmaf_rn(dx, -theta, X.z);
        X.z = K == 0 ? X.z : __saturatef(__fmaf_rn(X.w, -0x1p100f, ux));
        a.rec[0][r] = X;
        a.rec[1][r] = X;
        if (K >= 1) a.u[r] = ux;
    }
}

__global__ void __launch_bounds__(256)
k_rdc_grp2(const RdcIter a, const int32_t *slots, const int32_t *lpos, int first1, int n1, int nb1,
           int first0, int n0) {
    __shared__ float sm[5 * 256];
    if ((int)blockIdx.x < nb1)
        grp_body2<256>(a, slots, lpos, first1, n1, blockIdx.x, sm);
    else
        grp_body2<32>(a, slots, lpos, first0, n0, blockIdx.x - nb1, sm);
}

__global__ void __launch_bounds__(1024)
k_rdc_grp2_big(const RdcIter a, const int32_t *slots, const int32_t *lpos, int first, int nslots) {
    __shared__ float sm[5 * 1024];
    grp_body2<1024>(a, slots, lpos, first, nslots, blockIdx.x, sm);
}

// one launch for the 256-thread blocks: the first nb1 CTAs run segment 1 (components of 64 ..
// 256 records, CTA barrier), the rest segment 0 (eight independent warp blocks per CTA)
#ifndef RDS_GRP_MINB
#define RDS_GRP_MINB 1  // resident 256-thread CTAs per SM asked of the compiler (A/B: r02s2h)
#endif
__global__ void __launch_bounds__(256, RDS_GRP_MINB)
k_rdc_grp(const RdcIter a, const int32_t *slots, const int32_t *lpos, int first1, int n1, int nb1,
          int first0, int n0) {
    __shared__ float4 sm[2][256];
    if ((int)blockIdx.x < nb1)
        grp_body<256>(a, slots, lpos, first1, n1, blockIdx.x, sm);
    else
        grp_body<32>(a, slots, lpos, first0, n0, blockIdx.x - nb1, sm);
}

__global__ void __launch_bounds__(1024)
k_rdc_grp_big(const RdcIter a, const int32_t *slots, const int32_t *lpos, int first, int nslots) {
    __shared__ float4 sm[2][1024];
    grp_body<1024>(a, slots, lpos, first, nslots, blockIdx.x, sm);
}

}  // namespace

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// CTA sum of two doubles in a fixed order (xor-shuffle tree, then the warps in order); the
// result is valid in thread 0
__device__ __forceinline__ void cta_sum2(double &a, double &b, double (*sh)[RDC_THREADS / 32]) {
    a = warp_sum_d(a);
    b = warp_sum_d(b);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        sh[0][w] = a;
        sh[1][w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a = b = 0.0;
        for (int i = 0; i < RDC_THREADS / 32; ++i) {
            a += sh[0][i];
            b += sh[1][i];
        }
    }
}

// Each CTA owns a contiguous range of RD pixels (neighbours in the row above / below are
// nearby records: L1 reuse).  NPT > 0: every thread owns the fixed pixels
// start + t + q * blockDim (q < NPT) and keeps their codes in registers for the whole solve;
// NPT = 0: any n, codes reloaded every pass.
// Cluster form for small bands (CL): the whole grid is ONE thread-block cluster (<= 16 CTAs,
// one per SM), so the per-iteration barrier is the hardware cluster barrier (release /
// acquire at cluster scope) instead of the global-memory grid barrier.
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Neighbour synchronisation (NB form, fixed-K solves): instead of a grid barrier, a CTA
// publishes "pass k done" in its own counter (release) and, before pass k + 1, waits only for
// the CTAs that own records its pixels read (acquire).  The owner relation is symmetric (the
// six stencil neighbours come in pairs up/down, ur/dl, left/right), so the same wait also
// guarantees that those CTAs have finished READING this CTA's records of pass k before pass
// k + 1 overwrites that ping-pong buffer, and any two CTAs that read a common record are at
// most one pass apart -- they then read different buffers.  Ranges are whole 128-byte lines
// of records (multiples of 8), so no L1 line mixes two CTAs' records either: a line that
// another CTA of the same SM brings into L1 holds the data of the pass this CTA reads or of
// the other buffer, never a stale copy of the same one.
__device__ __forceinline__ void nbr_sync(int *prog, int lo, int hi, int k1) {
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(prog + blockIdx.x), "r"(k1)
                     : "memory");
    const int c = lo + (int)threadIdx.x;
    if (c <= hi && c != (int)blockIdx.x) {
        // spin relaxed (an acquire load also invalidates the SM's L1, which the CTAs still
        // computing on this SM depend on), then one acquire once the count is reached
        int v;
        do {
            asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(prog + c)
                         : "memory");
        } while (v < k1);
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(prog + c) : "memory");
    }
    __syncthreads();
}

template <int NPT, bool CL = false, bool NB = false>
__global__ void __launch_bounds__(RDC_THREADS) k_rdc_iter(const RdcIter a) {
    // (NB: CTA ranges of whole 128-byte record lines)
    const int chunk = NB ? (((a.n + gridDim.x - 1) / gridDim.x + 7) & ~7)
                         : (a.n + gridDim.x - 1) / gridDim.x;
    const int start = blockIdx.x * chunk;
    const int stop = min(a.n, start + chunk);
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    uint2 cw[NPT > 0 ? NPT : 1];  // packed codes of the owned pixels (2 registers each)
    int ri[NPT > 0 ? NPT : 1];    // their record indices (-1: none)
    const int32_t *sel = a.sel;   // the coupled pixels of a split solve, else every record
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
        const int i = start + threadIdx.x + q * blockDim.x;
        ri[q] = i < stop ? (sel ? __ldg(sel + i) : i) : -1;
        cw[q] = ri[q] >= 0 ? __ldg(a.code + ri[q]) : make_uint2(0u, 0u);
    }
    __shared__ double sh[2][RDC_THREADS / 32];
    __shared__ int stop_s;
    // NB: the CTAs owning a record some pixel of this CTA reads (always including itself)
    int dep_lo = blockIdx.x, dep_hi = blockIdx.x;
    int *prog = reinterpret_cast<int *>(reinterpret_cast<char *>(a.bar) + 128);
    if (NB) {
        __shared__ int s_lo, s_hi;
        if (threadIdx.x == 0) {
            s_lo = a.n;
            s_hi = -1;
        }
        __syncthreads();
        int lo = a.n, hi = -1;
        for (int r = start + threadIdx.x; r < stop; r += blockDim.x) {
            const PixConst q = decode(__ldg(a.code + r), r);
            const int nb[6] = {q.up, q.ur, q.lf, q.dn, q.dl, q.rt};
#pragma unroll
            for (int e = 0; e < 6; ++e)
                if (nb[e] >= 0) {
                    lo = min(lo, nb[e]);
                    hi = max(hi, nb[e]);
                }
        }
        atomicMin(&s_lo, lo);
        atomicMax(&s_hi, hi);
        __syncthreads();
        if (s_hi >= 0) {
            dep_lo = min(dep_lo, s_lo / chunk);
            dep_hi = max(dep_hi, s_hi / chunk);
        }
    }
    const int m = a.check_every;  // tolerance solves: check after iterations m, 2m, ..., K
    int nchk = 0;                 // checks so far: selects the partial-sum buffer
    for (int k = 0; k <= a.K; ++k) {
        const bool odd = k & 1;  // selects: a runtime index into a.rec would cost a stack copy
        const float4 *B = odd ? a.rec[1] : a.rec[0];
        float4 *O = odd ? a.rec[0] : a.rec[1];
        const bool chk = m > 0 && k >= 1 && (k % m == 0 || k == a.K);
        const bool chk_next = m > 0 && k + 1 <= a.K && ((k + 1) % m == 0 || k + 1 == a.K);
        const bool wr_u = k >= 1 && (k == a.K || chk || chk_next);
        float su = 0.0f, sv = 0.0f;
        if (NPT > 0) {
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                if (ri[q] >= 0)
                    pix_pass(decode(cw[q], ri[q]), B, O, a.u, k, a.K, tau, theta, inv_theta,
                             chk, wr_u, su, sv);
            }
        } else {
            for (int i = start + threadIdx.x; i < stop; i += blockDim.x) {
                const int r = sel ? __ldg(sel + i) : i;
                pix_pass(decode(__ldg(a.code + r), r), B, O, a.u, k, a.K, tau, theta,
                         inv_theta, chk, wr_u, su, sv);
            }
        }
        // two buffers alternating by check parity: when checks are one pass apart no barrier
        // separates a fast CTA's write for check c+1 from a slow CTA's read for check c
        double *part = a.part + (nchk & 1) * 2 * RDC_MAX_GRID;
        if (chk) {  // this CTA's partial sums, published by the barrier below
            double du = su, dv = sv;
            cta_sum2(du, dv, sh);
            if (threadIdx.x == 0) {
                part[2 * blockIdx.x] = du;
                part[2 * blockIdx.x + 1] = dv;
            }
            ++nchk;
        }
        if (k < a.K || m > 0) {
            if (CL)
                cluster_barrier();
            else if (NB)
                nbr_sync(prog, dep_lo, dep_hi, k + 1);
            else
                grid_barrier(a.bar, (unsigned long long)(k + 1));
        }
        if (chk) {  // every CTA forms the same total in the same order: one common decision
            double tu = 0.0, tv = 0.0;
            for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
                tu += __ldcg(part + 2 * b);
                tv += __ldcg(part + 2 * b + 1);
            }
            cta_sum2(tu, tv, sh);
            if (threadIdx.x == 0) {
                const double r = fmax(sqrt(tu / a.norm_div), sqrt(tv / a.norm_div));
                const bool conv = r <= a.tol, fire = conv || k == a.K;
                stop_s = fire;
                if (blockIdx.x == 0) {
                    StopRecord *rec = a.rec_out;
                    rec->residual = r;
                    rec->checks += 1;
                    rec->it = k;
                    if (fire) {
                        rec->iters = k;
                        rec->converged = conv ? 1 : 0;
                        rec->launches = 0;
                        rec->flag = 1;
                    }
                }
            }
            __syncthreads();
            if (stop_s) break;
        }
    }
}

typedef void (*RdcFn)(const RdcIter);

template <int NPT>
static int grid_of(int n_sm) {
    static int b = 0;
    if (b <= 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_rdc_iter<NPT>, RDC_THREADS, 0) !=
                cudaSuccess ||
            b < 1) {
            (void)cudaGetLastError();
            b = 1;
        }
        static const int cap = getenv("RDS_RDC_MAXB") ? atoi(getenv("RDS_RDC_MAXB")) : 3;
        if (b > cap) b = cap;  // fewer CTAs: a cheaper grid barrier (3 per SM: inside the bench
                               // C3 delta = .1 runs 14.5-14.7 ms vs 15.2 at 2 per SM, although
                               // the stand-alone sweep favoured 2; profiles/r02/r02al_*)
    }
    return b * n_sm;
}

cudaError_t launch_rdc_count(const uint8_t *lab, int64_t pitch, int H, int W, int32_t *rowcnt,
                             int32_t *rowoff, int32_t *total, cudaStream_t s) {
    const int g = (H + 7) / 8;
    k_rdc_rowcount<<<g, 256, 0, s>>>(lab, pitch, H, W, rowcnt);
    k_rdc_scan<<<1, 1024, 0, s>>>(rowcnt, H, rowoff, total);
    return cudaGetLastError();
}

cudaError_t launch_rdc_fill(const uint8_t *lab, int64_t pitch, int H, int W,
                            const int32_t *rowoff, int32_t *idxmap, int32_t *list,
                            cudaStream_t s) {
    k_rdc_fill<<<(H + 7) / 8, 256, 0, s>>>(lab, pitch, H, W, rowoff, idxmap, list);
    return cudaGetLastError();
}

cudaError_t launch_rdc_gather(const RdcSetup &a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    int g = (a.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_rdc_gather<<<g, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_rdc_scatter(const RdcSetup &a, const RdcIter &it, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    int g = (a.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_rdc_scatter<<<g, 256, 0, s>>>(a, it.rec[0], it.rec[1], it.K,
                                    it.check_every > 0 ? it.rec_out : nullptr);
    return cudaGetLastError();
}

cudaError_t launch_rdc_split(const uint2 *code, int n, int32_t *cnt, int32_t *off,
                             int32_t *n_cpl, int32_t *cpl, int32_t *iso, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int nb = (n + SPLIT_CHUNK - 1) / SPLIT_CHUNK;
    k_rdc_split_count<<<nb, SPLIT_CHUNK, 0, s>>>(code, n, cnt);
    k_rdc_scan<<<1, 1024, 0, s>>>(cnt, nb, off, n_cpl);
    k_rdc_split_fill<<<nb, SPLIT_CHUNK, 0, s>>>(code, n, off, cpl, iso);
    return cudaGetLastError();
}

cudaError_t launch_rdc_iso(const RdcIter &a, const int32_t *iso, int n_iso, int n_sm,
                           cudaStream_t s) {
    if (n_iso <= 0) return cudaSuccess;
    int g = (n_iso + 255) / 256;
    if (g > n_sm * 8) g = n_sm * 8;
    k_rdc_iso<<<g, 256, 0, s>>>(a, iso, n_iso);
    return cudaGetLastError();
}

cudaError_t launch_grp_label(const uint2 *code, const int32_t *cpl, int nc, int32_t *lab,
                             int32_t *cnt, int32_t *bad, int32_t *rank, int32_t *cidx,
                             int32_t *ctr, int *rounds, cudaStream_t s) {
    *rounds = 0;
    if (nc <= 0) return cudaSuccess;
    int g = (nc + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(int32_t) * 16, s);
    if (e != cudaSuccess) return e;
    k_grp_init<<<g, 256, 0, s>>>(cpl, nc, lab, cnt, bad, cidx);
    // rounds in batches of GRP_BATCH with one flag read-back each, until a batch's last round
    // lowers nothing (scattered noise bands: one or two batches) or GRP_ROUNDS_MAX is reached
    // (a band with long connected runs: the unsettled components then stay on the barrier)
    for (int p = 0; p < GRP_ROUNDS_MAX; p += GRP_BATCH) {
        for (int b = 0; b < GRP_BATCH - 1; ++b) k_grp_prop<<<g, 256, 0, s>>>(code, cpl, nc, lab, ctr + 13);
        e = cudaMemsetAsync(ctr + 12, 0, sizeof(int32_t), s);
        if (e != cudaSuccess) return e;
        k_grp_prop<<<g, 256, 0, s>>>(code, cpl, nc, lab, ctr + 12);
        int32_t changed = 0;
        e = cudaMemcpyAsync(&changed, ctr + 12, sizeof changed, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return e;
        e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return e;
        *rounds += GRP_BATCH;
        if (!changed) break;
    }
    k_grp_count<<<g, 256, 0, s>>>(code, cpl, nc, lab, cnt, bad, rank);
    k_grp_class<<<(nc + 255) / 256, 256, 0, s>>>(cpl, nc, lab, cnt, bad, cidx, ctr);
    return cudaGetLastError();
}

// slot layout from the class counts ctr[1..10]: segment 0 = classes 32 .. 2 (warp blocks),
// 1 = 256 .. 64, 2 = 1024, 512; every segment starts on a multiple of 1024 and holds its
// classes by falling size, so each 2^k range is aligned to 2^k
void grp_layout(const int32_t *ctr, GrpPlan *gp) {
    static const int seg_hi[3] = {5, 8, 10}, seg_lo[3] = {1, 6, 9};
    int pos = 0;
    for (int sg = 0; sg < 3; ++sg) {
        gp->first[sg] = pos;
        for (int k = seg_hi[sg]; k >= seg_lo[sg]; --k) {
            gp->base[k] = pos;
            pos += ctr[k] << k;
        }
        gp->count[sg] = pos - gp->first[sg];
        pos = (pos + 1023) & ~1023;
    }
    gp->total = pos;
}

cudaError_t launch_grp_fill(const int32_t *cpl, int nc, const int32_t *lab, const int32_t *cidx,
                            const int32_t *rank, const GrpPlan &gp, int32_t *slots,
                            int32_t *lpos, int32_t *fb, int32_t *nfb, cudaStream_t s) {
    if (nc <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(slots, 0xff, sizeof(int32_t) * (size_t)(gp.total > 0 ? gp.total : 1), s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(nfb, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    GrpBases gb;
    for (int k = 0; k < 11; ++k) gb.base[k] = gp.base[k];
    int g = (nc + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_grp_fill<<<g, 256, 0, s>>>(cpl, nc, lab, cidx, rank, gb, slots, lpos, fb, nfb);
    return cudaGetLastError();
}

cudaError_t launch_rdc_grp(const RdcIter &a, const GrpPlan &gp, const int32_t *slots,
                           const int32_t *lpos, cudaStream_t s) {
    static const bool two_phase = [] {
        const char *e = getenv("RDS_GRP_2PH");
        return e ? atoi(e) != 0 : GRP_2PH_DEFAULT;
    }();
    const int nb0 = (gp.count[0] + 255) / 256, nb1 = (gp.count[1] + 255) / 256;
    const int nb2 = (gp.count[2] + 1023) / 1024;
    if (nb0 + nb1 > 0) {
        if (two_phase)
            k_rdc_grp2<<<nb0 + nb1, 256, 0, s>>>(a, slots, lpos, gp.first[1], gp.count[1], nb1,
                                                 gp.first[0], gp.count[0]);
        else
            k_rdc_grp<<<nb0 + nb1, 256, 0, s>>>(a, slots, lpos, gp.first[1], gp.count[1], nb1,
                                                gp.first[0], gp.count[0]);
    }
    if (nb2 > 0) {
        if (two_phase)
            k_rdc_grp2_big<<<nb2, 1024, 0, s>>>(a, slots, lpos, gp.first[2], gp.count[2]);
        else
            k_rdc_grp_big<<<nb2, 1024, 0, s>>>(a, slots, lpos, gp.first[2], gp.count[2]);
    }
    return cudaGetLastError();
}

// Can one cluster of g CTAs of fn be scheduled on this device (a g > 8 cluster needs the
// non-portable size; MIG / MPS slices or small GPCs may not hold it)?  Cached per (fn, g).
static bool cluster_fits(RdcFn fn, int npt_slot, int g) {
    static signed char ok[2][RDC_CLUSTER_MAX + 1];  // 0 unknown, 1 yes, -1 no
    signed char &c = ok[npt_slot][g];
    if (c == 0) {
        bool fits = true;
        if (g > 8 && cudaFuncSetAttribute((const void *)fn,
                                          cudaFuncAttributeNonPortableClusterSizeAllowed,
                                          1) != cudaSuccess)
            fits = false;
        if (fits) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(g);
            cfg.blockDim = dim3(RDC_THREADS);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = g;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = 0;
            fits = cudaOccupancyMaxActiveClusters(&n, (const void *)fn, &cfg) == cudaSuccess &&
                   n >= 1;
        }
        (void)cudaGetLastError();
        c = fits ? 1 : -1;
    }
    return c > 0;
}

// one cluster of g CTAs (g <= RDC_CLUSTER_MAX), NPT pixels per thread
static cudaError_t launch_cluster(const RdcIter &a, RdcFn fn, int g, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(RDC_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = g;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {const_cast<RdcIter *>(&a)};
    return cudaLaunchKernelExC(&cfg, (const void *)fn, args);
}

cudaError_t launch_rdc_iter(const RdcIter &a, int n_sm, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    static const bool use_cluster = !getenv("RDS_RDC_CLUSTER") || atoi(getenv("RDS_RDC_CLUSTER"));
    if (use_cluster && a.n <= RDC_CLUSTER_MAX * RDC_THREADS * 2) {
        const int npt = a.n <= RDC_CLUSTER_MAX * RDC_THREADS ? 1 : 2;
        const int g = (a.n + RDC_THREADS * npt - 1) / (RDC_THREADS * npt);
        RdcFn cf = npt == 1 ? k_rdc_iter<1, true> : k_rdc_iter<2, true>;
        // not schedulable as one cluster here: fall through to the cooperative grid form
        if (cluster_fits(cf, npt - 1, g)) return launch_cluster(a, cf, g, s);
    }
    // the smallest register-resident variant that covers n, else the general one.  RDS_RDC_NB=1:
    // fixed-K solves synchronise with their neighbour CTAs only (NB form; off by default:
    // measured 3% faster at C3 delta = .1 but 1.3-4x slower at thinner bands)
    static const bool nb_env = getenv("RDS_RDC_NB") && atoi(getenv("RDS_RDC_NB"));
    // (NB needs both record buffers on 128-byte lines: ranges of whole lines, see nbr_sync)
    const bool nb = nb_env && a.check_every <= 0 && !a.sel && (a.rec[1] - a.rec[0]) % 8 == 0 &&
                    (reinterpret_cast<uintptr_t>(a.rec[0]) & 127) == 0;
    RdcFn fn = nullptr;
    int g = 0;
    const int64_t n = a.n;
    static const int max_npt = getenv("RDS_RDC_MAXNPT") ? atoi(getenv("RDS_RDC_MAXNPT")) : 2;
    if (n <= (int64_t)grid_of<1>(n_sm) * RDC_THREADS) {
        fn = nb ? k_rdc_iter<1, false, true> : k_rdc_iter<1>;
        g = grid_of<1>(n_sm);
    } else if (max_npt >= 2 && n <= (int64_t)grid_of<2>(n_sm) * RDC_THREADS * 2) {
        fn = nb ? k_rdc_iter<2, false, true> : k_rdc_iter<2>;
        g = grid_of<2>(n_sm);
    } else if (max_npt >= 4 && n <= (int64_t)grid_of<4>(n_sm) * RDC_THREADS * 4) {
        fn = nb ? k_rdc_iter<4, false, true> : k_rdc_iter<4>;
        g = grid_of<4>(n_sm);
    } else if (max_npt >= 8 && n <= (int64_t)grid_of<8>(n_sm) * RDC_THREADS * 8) {
        fn = nb ? k_rdc_iter<8, false, true> : k_rdc_iter<8>;
        g = grid_of<8>(n_sm);
    } else if (max_npt >= 16 && n <= (int64_t)grid_of<16>(n_sm) * RDC_THREADS * 16) {
        fn = nb ? k_rdc_iter<16, false, true> : k_rdc_iter<16>;
        g = grid_of<16>(n_sm);
    } else {
        fn = nb ? k_rdc_iter<0, false, true> : k_rdc_iter<0>;
        g = grid_of<0>(n_sm);
    }
    const int64_t need = (n + RDC_THREADS - 1) / RDC_THREADS;
    if (g > need) g = (int)need;
    if (g > RDC_MAX_GRID) g = RDC_MAX_GRID;
    if (nb) {  // ranges of whole 8-record lines: no more CTAs than ranges
        const int64_t per = ((n + g - 1) / g + 7) & ~7;
        g = (int)((n + per - 1) / per);
    }
    void *args[] = {const_cast<RdcIter *>(&a)};
    cudaError_t e = cudaMemsetAsync(a.bar, 0, RDC_BAR_BYTES, s);
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel((const void *)fn, dim3(g), dim3(RDC_THREADS), args, 0, s);
}

}  // namespace rds
