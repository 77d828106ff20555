// k_stencil.cu -- K3, the hot loop of librds: S fused outer iterations of the restricted-
// domain dual iteration per HBM round trip (temporal blocking), sm_100a.
//
// One outer iteration (PAPER.md:58-70 alternation, restricted forms Eq. 7-9):
//   w   = div rho - v/theta                                   (reading R-C5)
//   rho = (rho + tau grad w) / (1 + tau |grad w|) on RD, 0 on Fg u Bg
//   u   = v - theta div rho on RD, u0 elsewhere
//   v   = min(max(u - theta lambda f, 0), 1) on RD, u0 elsewhere
// with grad = forward differences (zero on row H-1 / column W-1) and div = -grad^T
// (reading R-C6).  The label and theta*lambda*f are folded into one float c per pixel:
// c = theta*lambda*f on RD, -inf on Fg, +inf on Bg and on the frame, so
// sat(u - c) (FADD.SAT) reproduces the pinned u0 exactly, and |c| * 2^-120 under the
// square root of |grad w| makes rho's update factor exactly 0 off RD.
//
// Execution model.  Each warp owns one work item: a strip of 128 columns
// (4 per lane, float4 loads/stores, 512 B per row per array) of which WV = wv_of(KF) are
// output columns, marching down the rows of a chunk.  The S iterations are a software
// pipeline in registers: stage t consumes level t-1 at row m+1 and emits level t at row m,
// so each input row is read once from HBM and each output row written once per S
// iterations.  Horizontal neighbours come from warp shuffles (2 per stage per row); the
// dependency cone (KF+1 columns/rows behind, KF ahead) is recomputed redundantly at the
// strip and chunk edges instead of being exchanged.
//
// Stage state per pixel (level t-1 at the stage's row m): rho1, rho2, v, c, w.  rho1 of
// level t at row m-1 (needed by div) is the next stage's rho1 state, so it is not stored
// twice.  The row loop is unrolled by two with two state sets (A -> B, B -> A) so the
// per-row state shift is register renaming, not moves.
#include <math.h>

#include "internal.h"

namespace rds {

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void st4(float *p, const float (&x)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Input rows are staged in shared memory with cp.async (LDGSTS): a RING of slots per warp
// for rho1, rho2, v (3 planes x 32 lanes x float4 = 1.5 KB per row) and a c ring that every
// stage re-reads at its own (lagging) row instead of carrying c in registers.  The c ring
// keeps each row twice (slots r mod CR and r mod CR + CR), so the row n-L of stage t is at a
// compile-time offset -L from row n's upper copy: no index arithmetic per stage.  Every lane
// copies and later reads only its own 16-byte pieces, so no cross-lane synchronisation is
// needed (cp.async.wait_group is per-thread).
constexpr int RING = 4;   // rows of rho1/rho2/v in flight (power of two)
constexpr int CR = 16;    // rows of c kept (power of two; >= RING + KF + 3)
constexpr int STENCIL_SMEM = STENCIL_WARPS * (RING * 96 + 2 * CR * 32) * (int)sizeof(float4);

// Pipeline split: stages [0, SPLIT) and [SPLIT, S) are joined through a one-row delay
// buffer D, so within one row step the two halves are independent dependency chains (twice
// the instruction-level parallelism for 16 extra registers).
template <int S>
struct Split {
    static constexpr int value = S >= 4 ? S / 2 : 0;
};

template <int S>
struct PipeState {
    float p1[S][4], p2[S][4], v[S][4], w[S][4];
    float q1[4];                       // rho1 of the last level at the previous emitted row
    float d1[4], d2[4], dv[4], dd[4];  // delay buffer (level SPLIT output, one row back)
};

struct Ctx {
    const float *p1i, *p2i, *vi, *ci;
    float *p1o, *p2o, *vo, *uo;
    uint8_t *mo;
    float4 *ring;   // this lane's slot 0, plane 0; slot stride 96 float4, plane stride 32
    float4 *cring;  // this lane's c slot 0; slot stride 32 float4, 2*CR slots
    int64_t pitch;
    int col, H, R0, Rend, n_last;
    bool store_lane, right_edge;
    float kx[4];
    float tau, theta, inv_theta;
};

__device__ __forceinline__ void stage_row(const Ctx &x, int r) {
    const int rr = r & (RING - 1);  // two's complement: also right for r < 0
    const int rc = r & (CR - 1);
    float4 *slot = x.ring + rr * 96;
    const int64_t off = (int64_t)r * x.pitch;
    cp_async16(slot, x.p1i + off);
    cp_async16(slot + 32, x.p2i + off);
    cp_async16(slot + 64, x.vi + off);
    cp_async16(x.cring + rc * 32, x.ci + off);
    cp_async16(x.cring + (rc + CR) * 32, x.ci + off);
}

// One stage: consumes level t at row m+1 (in1, in2, inv and ind = div rho there, computed
// once by the stage that emitted the row), uses the stage state (level t at row m) and q1
// (rho1 of level t+1 at row m-1), emits level t+1 at row m (o1, o2, ov, od) and the new
// state (level t at row m+1).
template <bool WRITE_U, bool ALIGNED, bool LAST>
__device__ __forceinline__ void stage(const float (&ap1)[4], const float (&ap2)[4],
                                      const float (&av)[4], const float (&aw)[4],
                                      const float (&q1)[4], const float (&in1)[4],
                                      const float (&in2)[4], const float (&inv)[4],
                                      const float (&ind)[4], const float4 &c4, int m,
                                      const Ctx &x,
                                      float (&bp1)[4], float (&bp2)[4], float (&bv)[4],
                                      float (&bw)[4], float (&o1)[4], float (&o2)[4],
                                      float (&ov)[4], float (&od)[4], float (&ou)[4]) {
    constexpr unsigned FULL = 0xffffffffu;
    const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
    float w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)  // w at row m+1; ind = div rho there (from the emitter)
        w[e] = fmaf(inv[e], -x.inv_theta, ind[e]);
    float wr = __shfl_down_sync(FULL, aw[0], 1);
    if (ALIGNED && x.right_edge) wr = aw[3];       // grad_2 = 0 on column W-1
    const bool last_row = LAST && (m == x.H - 1);  // grad_1 = 0 on row H-1
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // rho-step at row m
        float g1 = w[e] - aw[e];
        if (LAST) g1 = last_row ? 0.0f : g1;
        float g2 = (e < 3 ? aw[e + 1] : wr) - aw[e];
        if (!ALIGNED) g2 *= x.kx[e];
        // rho = 0 off RD without predicates: c = +-inf there, so |c| * 2^-120 = inf enters
        // the square root and rr = 1 / (1 + tau inf) = 0.  On RD |c| <= 2^20 (clamped in K1),
        // so the added |c| * 2^-120 <= 2^-100 is far below float32 resolution of g^2 + ...
        const float e_rd = fabsf(cc[e]) * 0x1p-120f;
        const float rr =
            rcp_approx(fmaf(x.tau, sqrt_approx(fmaf(g1, g1, fmaf(g2, g2, e_rd))), 1.0f));
        o1[e] = fmaf(x.tau, g1, ap1[e]) * rr;
        o2[e] = fmaf(x.tau, g2, ap2[e]) * rr;
    }
    const float ol2 = __shfl_up_sync(FULL, o2[3], 1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {  // u-step and v-step at row m
        const float d = (o1[e] - q1[e]) + (o2[e] - (e ? o2[e - 1] : ol2));
        od[e] = d;  // div rho of level t+1 at row m: the next stage's w needs exactly this
        const float u = fmaf(-x.theta, d, av[e]);
        ov[e] = __saturatef(u - cc[e]);
        if (WRITE_U) ou[e] = (fabsf(cc[e]) < INFINITY) ? u : av[e];
        bp1[e] = in1[e];
        bp2[e] = in2[e];
        bv[e] = inv[e];
        bw[e] = w[e];
    }
}

// One row step: consume input row n from the ring, advance all S stages, store the level-S
// row if it is an output row of this item, then refill the slot with row n+RING.
template <int S, bool WRITE_U, bool ALIGNED, bool LAST>
__device__ __forceinline__ void pipe_step(const PipeState<S> &A, PipeState<S> &B, int n,
                                          const Ctx &x) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int SP = Split<S>::value;
    cp_async_wait<RING - 1>();
    const float4 *slot = x.ring + (n & (RING - 1)) * 96;
    const float4 *crow = x.cring + ((n & (CR - 1)) + CR) * 32;  // row n; row n-L at -32 L
    const float4 c1 = slot[0], c2 = slot[32], cv = slot[64];
    float in1[4] = {c1.x, c1.y, c1.z, c1.w};
    float in2[4] = {c2.x, c2.y, c2.z, c2.w};
    float inv[4] = {cv.x, cv.y, cv.z, cv.w};
    // div rho of the incoming row (level 0): rho1 of row n-1 is stage 0's rho1 state
    float ind[4];
    {
        const float l2 = __shfl_up_sync(FULL, in2[3], 1);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            ind[e] = (in1[e] - A.p1[0][e]) + (in2[e] - (e ? in2[e - 1] : l2));
    }
    float uu[4];
#pragma unroll
    for (int t = 0; t < S; ++t) {
        const int m = n - t - 1 - (SP && t >= SP ? 1 : 0);  // row emitted (level t+1)
        if (SP && t == SP) {  // second chain starts from the delay buffer
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                B.d1[e] = in1[e];
                B.d2[e] = in2[e];
                B.dv[e] = inv[e];
                B.dd[e] = ind[e];
                in1[e] = A.d1[e];
                in2[e] = A.d2[e];
                inv[e] = A.dv[e];
                ind[e] = A.dd[e];
            }
        }
        float q1[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            q1[e] = (t == S - 1) ? A.q1[e]
                    : (SP && t == SP - 1) ? A.d1[e]
                                          : A.p1[(t + 1 < S) ? t + 1 : 0][e];
        float o1[4], o2[4], ov[4], od[4];
        const float4 c4 = crow[-32 * (n - m)];  // n - m is a compile-time lag
        stage<WRITE_U, ALIGNED, LAST>(A.p1[t], A.p2[t], A.v[t], A.w[t], q1, in1, in2, inv, ind,
                                      c4, m, x, B.p1[t], B.p2[t], B.v[t], B.w[t], o1, o2, ov, od,
                                      uu);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            in1[e] = o1[e];
            in2[e] = o2[e];
            inv[e] = ov[e];
            ind[e] = od[e];
        }
        if (t == S - 1) {
#pragma unroll
            for (int e = 0; e < 4; ++e) B.q1[e] = o1[e];
            if (x.store_lane && m >= x.R0 && m < x.Rend) {
                const int64_t o = (int64_t)m * x.pitch + x.col;
                st4(x.p1o + o, o1);
                st4(x.p2o + o, o2);
                st4(x.vo + o, ov);
                if (WRITE_U) {
                    st4(x.uo + o, uu);
                    *reinterpret_cast<uchar4 *>(x.mo + o) =
                        make_uchar4(uu[0] > 0.5f, uu[1] > 0.5f, uu[2] > 0.5f, uu[3] > 0.5f);
                }
            }
        }
    }
    // refill the slot just consumed (its values are in registers and already used)
    if (n + RING <= x.n_last) stage_row(x, n + RING);
    cp_async_commit();
}

template <int S, bool WRITE_U, bool ALIGNED, bool LAST>
__device__ __forceinline__ void march(const Ctx &x, int n) {
    PipeState<S> A, B;
#pragma unroll
    for (int t = 0; t < S; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) A.p1[t][e] = A.p2[t][e] = A.v[t][e] = A.w[t][e] = 0.0f;
#pragma unroll
    for (int e = 0; e < 4; ++e) A.q1[e] = A.d1[e] = A.d2[e] = A.dv[e] = A.dd[e] = 0.0f;
    for (; n <= x.n_last; n += 2) {
        pipe_step<S, WRITE_U, ALIGNED, LAST>(A, B, n, x);
        pipe_step<S, WRITE_U, ALIGNED, LAST>(B, A, n + 1, x);
    }
}

// Two CTAs (8 warps) per SM: shared memory (88 KB per CTA) and registers both allow 2.
template <int S>
struct MinBlocks {
    static constexpr int value = 2;
};

template <int KF, int S, bool WRITE_U, bool ALIGNED>
__global__ void __launch_bounds__(STENCIL_WARPS * 32, MinBlocks<S>::value)
    k_stencil(const StencilArgs a) {
    static_assert(S >= 1 && S <= KF && KF + 3 <= PAD_R, "stage count");
    static_assert(RING + KF + 3 <= CR, "c ring too short for the stage lags");
    constexpr int LH = lh_of(KF), WV = wv_of(KF);
    constexpr int SP = Split<S>::value;
    extern __shared__ float4 smem[];  // [warps][RING][3][32] then [warps][2 CR][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_items = *a.n_items;
    Ctx x;
    x.pitch = a.pitch;
    x.H = a.H;
    x.tau = a.tau;
    x.theta = a.theta;
    x.inv_theta = a.inv_theta;
    x.p1o = a.p1_out;
    x.p2o = a.p2_out;
    x.vo = a.v_out;
    x.uo = a.u_out;
    x.mo = a.mask_out;
    x.ring = smem + warp * RING * 96 + lane;
    x.cring = smem + STENCIL_WARPS * RING * 96 + warp * 2 * CR * 32 + lane;
    // persistent warps: fetch items from this launch's queue until it is drained
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(a.queue, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= n_items) break;  // warp-uniform
        const Item item = a.items[it];
        const int b0 = item.bands & 0xffff, b1 = item.bands >> 16;
        x.R0 = b0 * TILE_H;
        x.Rend = min(b1 * TILE_H, a.H);
        x.col = item.strip * WV - LH + 4 * lane;
        x.store_lane = (4 * lane >= LH) && (4 * lane < LH + WV);
        x.right_edge = (x.col + 3 == a.W - 1);
#pragma unroll
        for (int e = 0; e < 4; ++e) x.kx[e] = (x.col + e == a.W - 1) ? 0.0f : 1.0f;
        x.p1i = a.p1_in + x.col;
        x.p2i = a.p2_in + x.col;
        x.vi = a.v_in + x.col;
        x.ci = a.c + x.col;
        // input rows [n, n_last]; the cone reaches S+1 rows up and S rows down, the delay
        // buffer adds one row of latency.  The step count is made even (one extra warm-up
        // row) for the two-state unrolled loop.
        x.n_last = x.Rend - 1 + S + (SP ? 1 : 0);
        int n = x.R0 - (S + 1);
        if (((x.n_last - n + 1) & 1) != 0) --n;
#pragma unroll
        for (int r = 0; r < RING; ++r) {
            if (n + r <= x.n_last) stage_row(x, n + r);
            cp_async_commit();
        }
        // the Neumann row H-1 matters whenever the march (cone included) reaches it
        if (x.n_last >= a.H - 1)
            march<S, WRITE_U, ALIGNED, true>(x, n);
        else
            march<S, WRITE_U, ALIGNED, false>(x, n);
        cp_async_wait<0>();
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------
// dispatch over (KF, S, WRITE_U, ALIGNED)
// ---------------------------------------------------------------------------------------
typedef void (*StencilFn)(const StencilArgs);

template <int KF, int S>
struct Table {
    static void fill(StencilFn (*t)[2][2]) {
        t[S][0][0] = k_stencil<KF, S, false, false>;
        t[S][1][0] = k_stencil<KF, S, true, false>;
        t[S][0][1] = k_stencil<KF, S, false, true>;
        t[S][1][1] = k_stencil<KF, S, true, true>;
        Table<KF, S - 1>::fill(t);
    }
};
template <int KF>
struct Table<KF, 0> {
    static void fill(StencilFn (*)[2][2]) {}
};

#define RDS_KF_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)

static const int kKfMax = 8;

static StencilFn lookup(int kf, int stages, bool write_u, bool aligned) {
    static StencilFn table[kKfMax + 1][kKfMax + 1][2][2];
    static bool init = false;
    if (!init) {
#define RDS_FILL(K) Table<K, K>::fill(table[K]);
        RDS_KF_LIST(RDS_FILL)
#undef RDS_FILL
        for (auto &a : table)
            for (auto &b : a)
                for (auto &c : b)
                    for (StencilFn f : c)
                        if (f)
                            cudaFuncSetAttribute((const void *)f,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 STENCIL_SMEM);
        init = true;
    }
    if (kf < 1 || kf > kKfMax || stages < 1 || stages > kf) return nullptr;
    return table[kf][stages][write_u ? 1 : 0][aligned ? 1 : 0];
}

bool kf_supported(int kf) { return lookup(kf, 1, false, false) != nullptr; }

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
    StencilFn fn = lookup(kf, stages, false, aligned);
    if (!fn) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, STENCIL_WARPS * 32,
                                                      STENCIL_SMEM) != cudaSuccess)
        return 0;
    return nb;
}

cudaError_t launch_stencil(int kf, int stages, bool write_u, const StencilArgs &a, int grid,
                           cudaStream_t s) {
    StencilFn fn = lookup(kf, stages, write_u, (a.W & 3) == 0);
    if (!fn) return cudaErrorInvalidValue;
    if (grid <= 0) return cudaSuccess;
    fn<<<grid, STENCIL_WARPS * 32, STENCIL_SMEM, s>>>(a);
    return cudaGetLastError();
}

}  // namespace rds
