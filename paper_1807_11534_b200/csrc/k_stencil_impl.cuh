// k_stencil_impl.cuh -- K3, the hot loop of librds (included by k_stencil.cu, the dispatch,
// and by the per-k_fuse instantiation units k_stencil_kf*.cu, which build in parallel):
// S fused outer iterations of the restricted-
// domain dual iteration per HBM round trip (temporal blocking), sm_100a.
//
// One outer iteration (PAPER.md:58-70 alternation, restricted forms Eq. 7-9):
//   w   = div rho - v/theta                                   (reading R-C5)
//   rho = (rho + tau grad w) / (1 + tau |grad w|) on RD, 0 on Fg u Bg
//   u   = v - theta div rho on RD, u0 elsewhere
//   v   = min(max(u - theta lambda f, 0), 1) on RD, u0 elsewhere
// with grad = forward differences (zero on row H-1 / column W-1) and div = -grad^T
// (reading R-C6).  The label and theta*lambda*f are folded into one float per pixel,
// c' = 2^-100 theta*lambda*f on RD, -inf on Fg, +inf on Bg and on the frame, so
// sat(u - c) = FFMA.SAT(c', -2^100, u) reproduces the pinned u0 exactly, and |c'| added
// under the square root of |grad w| makes rho's update factor exactly 0 off RD.
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
// All per-pixel arithmetic is packed f32x2 (FFMA2 / FADD2 / FMUL2) on quad-swizzled data
// (see "Packed-pair arithmetic" below); only the two MUFU ops and the saturating v-step are
// scalar.
//
// Stage state per pixel (level t-1 at the stage's row m): rho1, rho2, v, w.  rho1 of
// level t at row m-1 (needed by div) is the next stage's rho1 state, so it is not stored
// twice.  The row loop is unrolled by two with two state sets (A -> B, B -> A) so the
// per-row state shift is register renaming, not moves.
#pragma once
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

// ---------------------------------------------------------------------------------------
// Packed-pair arithmetic.  sm_100a issues FFMA2 / FADD2 / FMUL2 (PTX f32x2): one instruction
// does the same fp32 operation, with the same round-to-nearest result, on two lanes of a
// register pair.  The FMA pipe's lane throughput is unchanged (measured: FFMA2 issues at
// half the FFMA rate, scripts/micro/ffma2_tput.cu), but every packed op frees an issue slot,
// and this kernel is bound by instruction issue.
//
// A lane owns 4 consecutive columns x0..x3 of its strip.  The state planes rho1, rho2, v
// and c are stored QUAD-SWIZZLED in HBM (memory order x0 x2 x1 x3 within every aligned
// quad, internal.h), so one 16-byte load yields the pairs a = (x0, x2) and b = (x1, x3).
// With that pairing every horizontal difference is a pair op: x(j+1) - x(j) is b - a for
// the a pair and (x2, x4) - b for the b pair, where x2 = a.y and x4 comes from the next
// lane; the left neighbours for div are (x(-1), x1) and a.
// ---------------------------------------------------------------------------------------
struct Q {
    float2 a, b;  // a = (x0, x2), b = (x1, x3)
};
__device__ __forceinline__ float2 add2(float2 x, float2 y) { return __fadd2_rn(x, y); }
__device__ __forceinline__ float2 sub2(float2 x, float2 y) {
    return __fadd2_rn(x, make_float2(-y.x, -y.y));  // FADD2 with a negated operand
}
__device__ __forceinline__ float2 mul2(float2 x, float2 y) { return __fmul2_rn(x, y); }
__device__ __forceinline__ float2 mul2(float2 x, float s) { return __fmul2_rn(x, make_float2(s, s)); }
__device__ __forceinline__ float2 fma2(float2 x, float2 y, float2 z) { return __ffma2_rn(x, y, z); }
__device__ __forceinline__ float2 fma2(float2 x, float s, float2 z) {
    return __ffma2_rn(x, make_float2(s, s), z);
}
__device__ __forceinline__ float2 fma2(float2 x, float s, float t) {
    return __ffma2_rn(x, make_float2(s, s), make_float2(t, t));
}
__device__ __forceinline__ float2 absq(float2 x) {  // folds into the FFMA2 operand as |R|
    return make_float2(fabsf(x.x), fabsf(x.y));
}
__device__ __forceinline__ Q ldq(const float4 &m) {
    return Q{make_float2(m.x, m.y), make_float2(m.z, m.w)};
}
__device__ __forceinline__ void stq(float *p, const Q &x) {  // swizzled store
    *reinterpret_cast<float4 *>(p) = make_float4(x.a.x, x.a.y, x.b.x, x.b.y);
}
__device__ __forceinline__ Q zeroq() {
    return Q{make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
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
// Per warp after the row rings: its c ring (2 CR rows of 32 float4) followed by two rows of
// 32 float4, the wavefront's per-lane 32-byte slots (k_wave; WaveSlot).  CRW = that stride.
constexpr int CRW = 2 * CR * 32 + 64;
constexpr int STENCIL_SMEM = STENCIL_WARPS * (RING * 96 + CRW) * (int)sizeof(float4);

// Pipeline split: the S stages are cut into NS+1 chains ([0, sp(1)), [sp(1), sp(2)), ...)
// joined through one-row delay buffers, so within one row step the chains are independent
// dependency chains (instruction-level parallelism for 16 registers per extra chain).  Three
// chains for S >= 6 measured best (RDS_CHAINS overrides for experiments).
#ifndef RDS_CHAINS
#define RDS_CHAINS 3
#endif
template <int S>
struct Split {
    static constexpr int NS = S >= 3 * RDS_CHAINS - 3 && RDS_CHAINS >= 3 ? RDS_CHAINS - 1
                              : S >= 4                                 ? 1
                                                                       : 0;
    // k-th split point, k = 1..NS
    __host__ __device__ static constexpr int sp(int k) { return (k * S) / (NS + 1); }
    // number of split points <= t (the extra row lag of stage t)
    __host__ __device__ static constexpr int lag(int t) {
        int n = 0;
        for (int k = 1; k <= NS; ++k) n += sp(k) <= t;
        return n;
    }
    // k if t == sp(k), else 0
    __host__ __device__ static constexpr int at(int t) {
        for (int k = 1; k <= NS; ++k)
            if (sp(k) == t) return k;
        return 0;
    }
};

// Warm-up elision (the trapezoid of the vertical cone; the "prologue" kernels k_stencil_pro,
// DESIGN.md §5).  Level S is stored on rows [R0, Rend); one iteration reads rows m-1 .. m+1
// of rho and m .. m+1 of v, w (div rho at m needs rho1 at m-1), so level t is needed on rows
// >= R0 - 1 - (S - t) for rho and >= R0 - (S - t) for v.  Stage t emits level t+1 at row
// m = n - t - 1 - lag(t) in row step n, so its rows are needed from row step
// n = R0 - S + 2t + 1 + lag(t) on; before that it only carries its state (the row it received
// and its w) and passes its input through.  At the first active step the stage's own previous
// row (q1, rho1 of level t+1 at row m-1) is a placeholder, but it enters only v and div rho of
// level t+1 at row m, which are needed one row lower.
template <int S>
struct Act {
    // first row step (relative to R0) in which stage t does its work
    __host__ __device__ static constexpr int first(int t) { return 1 - S + 2 * t + Split<S>::lag(t); }
    // prologue length of a march starting at R0 - S - 2: until every stage is active, even
    __host__ __device__ static constexpr int prologue() { return ((first(S - 1) + S + 2) + 1) & ~1; }
};

template <int S>
struct PipeState {
    static constexpr int ND = Split<S>::NS > 0 ? Split<S>::NS : 1;
    Q p1[S], p2[S], v[S], w[S];
    Q q1;                                  // rho1 of the last level at the previous emitted row
    Q d1[ND], d2[ND], dv[ND], dd[ND];      // delay buffers (chain-boundary outputs, one row back)
};

struct Ctx {
    const float *p1i, *p2i, *vi, *ci;
    float *p1o, *p2o, *vo, *uo;
    uint8_t *mo;
    float4 *ring;   // this lane's slot 0, plane 0; slot stride 96 float4, plane stride 32
    float4 *cring;  // this lane's c slot 0; slot stride 32 float4, 2*CR slots
    int64_t pitch;
    int col, H, R0, Rend, n_last;
    int chk_r0, chk_r1;  // CHECK mode: rows whose stopping sums are accumulated
    bool store_lane, right_edge;
    Q kx;
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

// rr = 1 / (1 + tau sqrt(s)) per element: two MUFU ops each, the FMA in between packed.
__device__ __forceinline__ float2 rr_of(float2 s, float tau) {
    const float2 den = fma2(make_float2(sqrt_approx(s.x), sqrt_approx(s.y)), tau, 1.0f);
    return make_float2(rcp_approx(den.x), rcp_approx(den.y));
}

// div rho at the lane's quad from rho1 (this row and the row above) and rho2 (this row);
// the left neighbour of x0 is the previous lane's x3.
__device__ __forceinline__ Q div_q(const Q &p1, const Q &p1up, const Q &p2) {
    const float l2 = __shfl_up_sync(0xffffffffu, p2.b.y, 1);
    Q d;
    d.a = add2(sub2(p1.a, p1up.a), sub2(p2.a, make_float2(l2, p2.b.x)));
    d.b = add2(sub2(p1.b, p1up.b), sub2(p2.b, p2.a));
    return d;
}

// Front half of a stage: w at row m+1 from the incoming row (inv, ind = div rho there), the
// gradient at row m from the state w (aw), and rr = 1 / (1 + tau |grad w|).
struct Front {
    Q w, g1, g2, rr;
};
template <bool ALIGNED, bool LAST>
__device__ __forceinline__ Front front(const Q &aw, const Q &inv, const Q &ind, const Q &c, int m,
                                       const Ctx &x) {
    constexpr unsigned FULL = 0xffffffffu;
    Front f;
    f.w.a = fma2(inv.a, -x.inv_theta, ind.a);
    f.w.b = fma2(inv.b, -x.inv_theta, ind.b);
    float wr = __shfl_down_sync(FULL, aw.a.x, 1);  // x4 of this lane = x0 of the next
    if (ALIGNED && x.right_edge) wr = aw.b.y;      // grad_2 = 0 on an image's column W-1
    f.g1.a = sub2(f.w.a, aw.a);
    f.g1.b = sub2(f.w.b, aw.b);
    if (LAST && m == x.H - 1) f.g1 = zeroq();      // grad_1 = 0 on row H-1
    f.g2.a = sub2(aw.b, aw.a);
    f.g2.b = sub2(make_float2(aw.a.y, wr), aw.b);
    if (!ALIGNED) {
        f.g2.a = mul2(f.g2.a, x.kx.a);
        f.g2.b = mul2(f.g2.b, x.kx.b);
    }
    // |grad w|^2 + |c'|: |c'| is +inf off RD (rr = 0) and <= 2^-80 on RD (see stage())
    f.rr.a = rr_of(fma2(f.g1.a, f.g1.a, fma2(f.g2.a, f.g2.a, absq(c.a))), x.tau);
    f.rr.b = rr_of(fma2(f.g1.b, f.g1.b, fma2(f.g2.b, f.g2.b, absq(c.b))), x.tau);
    return f;
}

// Back half at row m: the rho update (Eq. 8 fixed point), then, with q1 = rho1 of the new
// level at row m-1, div rho (od, exactly what the next stage's w needs), the u-step (Eq. 7)
// and the v-step (Eq. 9).
template <bool WRITE_U>
__device__ __forceinline__ void back(const Q &g1, const Q &g2, const Q &rr, const Q &ap1,
                                     const Q &ap2, const Q &av, const Q &q1, const Q &c,
                                     const Ctx &x, Q &o1, Q &o2, Q &ov, Q &od, Q &ou) {
    o1.a = mul2(fma2(g1.a, x.tau, ap1.a), rr.a);
    o2.a = mul2(fma2(g2.a, x.tau, ap2.a), rr.a);
    o1.b = mul2(fma2(g1.b, x.tau, ap1.b), rr.b);
    o2.b = mul2(fma2(g2.b, x.tau, ap2.b), rr.b);
    od = div_q(o1, q1, o2);
    Q u;
    u.a = fma2(od.a, -x.theta, av.a);
    u.b = fma2(od.b, -x.theta, av.b);
    ov.a = make_float2(__saturatef(fmaf(c.a.x, -0x1p100f, u.a.x)),
                       __saturatef(fmaf(c.a.y, -0x1p100f, u.a.y)));
    ov.b = make_float2(__saturatef(fmaf(c.b.x, -0x1p100f, u.b.x)),
                       __saturatef(fmaf(c.b.y, -0x1p100f, u.b.y)));
    if (WRITE_U) {
        ou.a = make_float2(fabsf(c.a.x) < INFINITY ? u.a.x : av.a.x,
                           fabsf(c.a.y) < INFINITY ? u.a.y : av.a.y);
        ou.b = make_float2(fabsf(c.b.x) < INFINITY ? u.b.x : av.b.x,
                           fabsf(c.b.y) < INFINITY ? u.b.y : av.b.y);
    }
}

// One stage: consumes level t at row m+1 (in1, in2, inv and ind = div rho there, computed
// once by the stage that emitted the row), uses the stage state (level t at row m) and q1
// (rho1 of level t+1 at row m-1), emits level t+1 at row m (o1, o2, ov, od) and the new
// state (level t at row m+1).
//
// c is stored as c' = c * 2^-100 (K1; exact for |c| >= 2^-26, within 2^-50 absolute below):
// |c'| <= 2^-80 on RD (|c| <= 2^20) is far below the fp32 resolution of |grad w|^2 and +inf
// off RD, where adding it under the square root makes the rho update factor exactly 0
// (rho = 0 on Fg u Bg, Eq. 8) without predicates or extra instructions (|c'| is an FFMA2
// operand modifier); u - c = fma(c', -2^100, u) exactly, and FFMA.SAT reproduces the pinned
// 0 / 1 off RD (Eq. 9).
template <bool WRITE_U, bool ALIGNED, bool LAST>
__device__ __forceinline__ void stage(const Q &ap1, const Q &ap2, const Q &av, const Q &aw,
                                      const Q &q1, const Q &in1, const Q &in2, const Q &inv,
                                      const Q &ind, const float4 &c4, int m, const Ctx &x,
                                      Q &bp1, Q &bp2, Q &bv, Q &bw, Q &o1, Q &o2, Q &ov, Q &od,
                                      Q &ou) {
    const Q c = ldq(c4);
    const Front f = front<ALIGNED, LAST>(aw, inv, ind, c, m, x);
    back<WRITE_U>(f.g1, f.g2, f.rr, ap1, ap2, av, q1, c, x, o1, o2, ov, od, ou);
    bp1 = in1;
    bp2 = in2;
    bv = inv;
    bw = f.w;
}

// ---------------------------------------------------------------------------------------
// Temporal wavefront (k_wave, DESIGN.md §5 "wavefront"): ONE persistent launch runs many
// KF-iteration blocks of a fixed-K solve.  Task (b, s) = block b of strip s: a warp marches
// the strip's active runs top to bottom, reading level b*KF from ping-pong buffer (c0+b)&1 and
// writing level (b+1)*KF into the other.  Block b's row r of strip s may be read only after
// block b-1 has written it on strips s-1, s, s+1 (the 128 input columns span them), so every
// task publishes a progress counter (rows < P final) and waits on its three producers'
// counters before it stages a row.  Tasks are taken in (b, s) order from one queue, so a task
// waits only on tasks already taken by running warps: no deadlock, no co-residency needed.
// The waits also order the ping-pong reuse: block b+1 overwrites a row of block b's input
// only after block b has emitted rows far below it (its march consumed the row by then).
// Rows outside [0, H) are frame rows (never written) and rows between active runs hold pinned
// values in both buffers, so neither is waited for.  The hooks run once per two row steps at
// the march's loop head, so the pipeline body itself has no extra control flow.
// ---------------------------------------------------------------------------------------

// Registers of a wavefront task; the counter addresses live in the lane's shared-memory slot
// (WaveSlot, after the warp's c ring) to keep the pipeline free of spills.  Everything here is
// warp-uniform (every lane loads / stores the same addresses) and branch-free except for
// vote-controlled loops, so the pipeline's warp shuffles need no divergence handling.
// rows between progress publications (a gpu-scope fence each); RDS_WAVE_PUB overrides (even)
#ifndef RDS_WAVE_PUB
#define RDS_WAVE_PUB 16
#endif
constexpr int WAVE_PUB = RDS_WAVE_PUB;
static_assert(WAVE_PUB >= 2 && WAVE_PUB % 2 == 0, "publication interval");

struct Wave {
    int avail;  // rows < avail are final on all three producers
    int pend;   // producers' progress loaded at the previous check
};
struct WaveSlot {
    const int *pin[3];      // progress of the producers on strips s-1, s, s+1 (a cell holding
                            // INT_MAX where there is none)
    int *pout;              // this task's progress counter
    const uint32_t *bits;   // the strip's band bitmask (k_wave's run loop state, kept out of
    int pos, task;          // registers while the pipeline runs)
};
__device__ __forceinline__ WaveSlot *wave_slot(const Ctx &x) {
    // the warp's slot after its c ring (x.cring is this lane's float4 of the c ring's row 0)
    return reinterpret_cast<WaveSlot *>(x.cring + 2 * CR * 32 - (threadIdx.x & 31));
}
static_assert(sizeof(WaveSlot) <= 64 * sizeof(float4), "wave slot");

__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int wave_poll(const WaveSlot *w) {
    return min(ld_relaxed(w->pin[0]), min(ld_relaxed(w->pin[1]), ld_relaxed(w->pin[2])));
}

// Rows < v of this task are final: make the warp's stores visible at gpu scope, then publish
// (every lane fences its own stores and writes the same value to the same word).
__device__ __forceinline__ void wave_publish(const Ctx &x, int v) {
    __syncwarp();
#ifndef RDS_WAVE_NOFENCE  // (timing experiment only: without the fence the protocol is unsafe)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
    __syncwarp();
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(wave_slot(x)->pout), "r"(v)
                 : "memory");
}

// The slow path of wave_need: a producer is always a task taken earlier by a running warp, so
// this wait ends; the bound (~seconds) turns a broken invariant into a launch error instead of
// a hung GPU.  (Conditions through warp votes: the compiler then knows the loop is uniform.)
__device__ __forceinline__ int wave_spin(const WaveSlot *ws, int avail, int need) {
    for (unsigned spins = 0; __any_sync(0xffffffffu, need > avail); ++spins) {
        if (spins > (1u << 24)) __trap();
        __nanosleep(128);
        avail = max(avail, wave_poll(ws));
    }
    return avail;
}

// Before staging input rows <= r: wait until the producers have finalised them.  The poll
// issued at the previous check is consumed first (its L2 round trip overlapped two row steps of
// work); the data is then read with cp.async.cg from L2, where the producer's fence put it
// before the counter.  The copies are issued only after the counter value has been observed
// (they are control dependent on it).
__device__ __forceinline__ void wave_need(const Ctx &x, Wave &w, int r) {
    const int need = min(r + 1, x.H);  // rows >= H are frame rows: never written
    if (__all_sync(0xffffffffu, w.avail >= x.H)) return;
    const WaveSlot *ws = wave_slot(x);
    w.avail = max(w.avail, w.pend);
    w.pend = wave_poll(ws);
    if (__any_sync(0xffffffffu, need > w.avail)) w.avail = wave_spin(ws, w.avail, need);
}

// Launch modes: PLAIN iterates; WRITE_U also writes u and the mask of the last level
// (the last launch of a solve); CHECK additionally accumulates the paper's stopping
// quantities sum (u^l - u^(l-1))^2 and sum (v^l - v^(l-1))^2 over the item's output pixels
// (f2, rds_solve_tol).  u^(l-1) comes from stage S-2 one row step earlier,
// or, for a single-stage launch, from the u plane written by the previous launch.
enum { MODE_PLAIN = 0, MODE_WRITE_U = 1, MODE_CHECK = 2 };

template <int S, int MODE>
struct Extra {  // per-row-step state only the CHECK mode needs
    Q uprev;    // u of level S-1 (stage S-2's u) at the last stage's row
};

// One row step: consume input row n from the ring, advance all S stages, store the level-S
// row if it is an output row of this item, then refill the slot with row n+RING.
template <int S, int MODE, bool ALIGNED, bool LAST, bool WAVE, int KST = -1>
__device__ __forceinline__ void pipe_step(const PipeState<S> &A, PipeState<S> &B,
                                          const Extra<S, MODE> &EA, Extra<S, MODE> &EB, int n,
                                          const Ctx &x, float &acc_u, float &acc_v, Wave &wv) {
    using SPL = Split<S>;
    constexpr bool WRITE_U = MODE != MODE_PLAIN;
    cp_async_wait<RING - 1>();
    const float4 *slot = x.ring + (n & (RING - 1)) * 96;
    const float4 *crow = x.cring + ((n & (CR - 1)) + CR) * 32;  // row n; row n-L at -32 L
    Q in1 = ldq(slot[0]), in2 = ldq(slot[32]), inv = ldq(slot[64]);
    // div rho of the incoming row (level 0): rho1 of row n-1 is stage 0's rho1 state
    Q ind = div_q(in1, A.p1[0], in2);
    Q uu;
#pragma unroll
    for (int t = 0; t < S; ++t) {
        const int m = n - t - 1 - SPL::lag(t);  // row emitted (level t+1)
        Q o1, o2, ov, od;
        if (SPL::at(t)) {  // a new chain starts from its delay buffer
            const int k = SPL::at(t) - 1;
            B.d1[k] = in1;
            B.d2[k] = in2;
            B.dv[k] = inv;
            B.dd[k] = ind;
            in1 = A.d1[k];
            in2 = A.d2[k];
            inv = A.dv[k];
            ind = A.dd[k];
        }
        const Q &q1 = (t == S - 1)          ? A.q1
                      : SPL::at(t + 1)      ? A.d1[SPL::at(t + 1) > 0 ? SPL::at(t + 1) - 1 : 0]
                                            : A.p1[(t + 1 < S) ? t + 1 : 0];
        const float4 c4 = crow[-32 * (n - m)];  // n - m is a compile-time lag
        // prologue step KST >= 0 (row step n = R0 - S - 2 + KST, compile time): a stage still
        // above its cone (Act) is elided -- it carries its state and passes its input on
        if (KST < 0 || KST - (S + 2) >= Act<S>::first(t)) {
            stage<WRITE_U, ALIGNED, LAST>(A.p1[t], A.p2[t], A.v[t], A.w[t], q1, in1, in2, inv,
                                          ind, c4, m, x, B.p1[t], B.p2[t], B.v[t], B.w[t], o1,
                                          o2, ov, od, uu);
        } else {
            B.p1[t] = in1;
            B.p2[t] = in2;
            B.v[t] = inv;
            B.w[t].a = fma2(inv.a, -x.inv_theta, ind.a);  // (dead unless the stage starts next)
            B.w[t].b = fma2(inv.b, -x.inv_theta, ind.b);
            o1 = in1;
            o2 = in2;
            ov = inv;
            od = ind;
            uu = inv;
        }
        in1 = o1;
        in2 = o2;
        inv = ov;
        ind = od;
        if (MODE == MODE_CHECK && S >= 2 && t == S - 2) EB.uprev = uu;  // u^(l-1), row m
        if (t == S - 1) {
            B.q1 = o1;
            if (x.store_lane && m >= x.R0 && m < x.Rend) {
                const int64_t o = (int64_t)m * x.pitch + x.col;
                if (MODE == MODE_CHECK) {
                    Q up;
                    if (S >= 2) {
                        up = EA.uprev;
                    } else {  // single stage: u^(l-1) is in the u plane (natural order)
                        const float4 q = *reinterpret_cast<const float4 *>(x.uo + o);
                        up = Q{make_float2(q.x, q.z), make_float2(q.y, q.w)};
                    }
                    const float2 da = sub2(uu.a, up.a), db = sub2(uu.b, up.b);
                    const Q &av = A.v[S - 1];  // v^(l-1) at row m
                    const float2 ea = sub2(ov.a, av.a), eb = sub2(ov.b, av.b);
                    if (m >= x.chk_r0 && m < x.chk_r1) {  // the rows the sums cover
                        acc_u += (da.x * da.x + da.y * da.y) + (db.x * db.x + db.y * db.y);
                        acc_v += (ea.x * ea.x + ea.y * ea.y) + (eb.x * eb.x + eb.y * eb.y);
                    }
                }
                stq(x.p1o + o, o1);
                stq(x.p2o + o, o2);
                stq(x.vo + o, ov);
                if (WRITE_U) {  // u and the mask are natural-order planes
                    *reinterpret_cast<float4 *>(x.uo + o) =
                        make_float4(uu.a.x, uu.b.x, uu.a.y, uu.b.y);
                    *reinterpret_cast<uchar4 *>(x.mo + o) =
                        make_uchar4(uu.a.x > 0.5f, uu.b.x > 0.5f, uu.a.y > 0.5f, uu.b.y > 0.5f);
                }
            }
        }
    }
    // refill the slot just consumed (its values are in registers and already used); the
    // wavefront first waits until the producers have written that row
    if (n + RING <= x.n_last) {
        if (WAVE) wave_need(x, wv, n + RING);
        stage_row(x, n + RING);
    }
    cp_async_commit();
}

// The prologue: row steps K, K+1, ... < P of a march that starts at n = R0 - S - 2, unrolled
// (each step's set of live stages is a compile-time constant); P is even, so the state ends in
// A as after the loop's step pairs.
template <int S, int MODE, bool ALIGNED, int K, int P>
struct Prologue {
    __device__ static __forceinline__ void run(PipeState<S> &A, PipeState<S> &B,
                                               Extra<S, MODE> &EA, Extra<S, MODE> &EB, int n,
                                               const Ctx &x, float &acc_u, float &acc_v,
                                               Wave &wv) {
        pipe_step<S, MODE, ALIGNED, false, false, K>(A, B, EA, EB, n, x, acc_u, acc_v, wv);
        pipe_step<S, MODE, ALIGNED, false, false, K + 1>(B, A, EB, EA, n + 1, x, acc_u, acc_v,
                                                         wv);
        Prologue<S, MODE, ALIGNED, K + 2, P>::run(A, B, EA, EB, n + 2, x, acc_u, acc_v, wv);
    }
};
template <int S, int MODE, bool ALIGNED, int P>
struct Prologue<S, MODE, ALIGNED, P, P> {
    __device__ static __forceinline__ void run(PipeState<S> &, PipeState<S> &, Extra<S, MODE> &,
                                               Extra<S, MODE> &, int, const Ctx &, float &,
                                               float &, Wave &) {}
};

template <int S, int MODE, bool ALIGNED, bool LAST, bool WAVE, bool PRO = false>
__device__ __forceinline__ void march(const Ctx &x, int n, float &acc_u, float &acc_v,
                                      Wave &wv) {
    PipeState<S> A, B;
    Extra<S, MODE> EA, EB;
#pragma unroll
    for (int t = 0; t < S; ++t) A.p1[t] = A.p2[t] = A.v[t] = A.w[t] = zeroq();
    A.q1 = zeroq();
#pragma unroll
    for (int k = 0; k < PipeState<S>::ND; ++k) {
        A.d1[k] = A.d2[k] = A.dv[k] = A.dd[k] = zeroq();
    }
    EA.uprev = zeroq();
    if (PRO && !LAST && !WAVE) {  // run_item started the march at R0 - S - 2 for this
        Prologue<S, MODE, ALIGNED, 0, Act<S>::prologue()>::run(A, B, EA, EB, n, x, acc_u, acc_v,
                                                               wv);
        n += Act<S>::prologue();
    }
    for (int k = 0; n <= x.n_last; n += 2, ++k) {
        // wavefront: every second loop head, publish the rows emitted so far (rows < n - S -
        // NS of this item are final)
        if (WAVE && (k % (WAVE_PUB / 2)) == WAVE_PUB / 2 - 1)
            wave_publish(x, min(max(n - S - Split<S>::NS, x.R0), x.Rend));
        pipe_step<S, MODE, ALIGNED, LAST, WAVE>(A, B, EA, EB, n, x, acc_u, acc_v, wv);
        pipe_step<S, MODE, ALIGNED, LAST, WAVE>(B, A, EB, EA, n + 1, x, acc_u, acc_v, wv);
    }
}

// One item: output columns of `strip`, output rows [r0, r1), inputs from the planes p1i /
// p2i / vi (pixel (0,0) origins).  Sets up the lane geometry, stages the first RING rows and
// marches (S stages); returns with every cp.async group drained.
template <int KF, int S, int MODE, bool ALIGNED, bool WAVE, bool PRO = false>
__device__ __forceinline__ void run_item(Ctx &x, const StencilArgs &a, int strip, int r0, int r1,
                                         const float *p1i, const float *p2i, const float *vi,
                                         float &acc_u, float &acc_v, Wave &wv) {
    constexpr int LH = lh_of(KF), WV = wv_of(KF);
    const int lane = threadIdx.x & 31;
    x.R0 = r0;
    x.Rend = r1;
    x.col = strip * WV - LH + 4 * lane;
    x.store_lane = (4 * lane >= LH) && (4 * lane < LH + WV);
    // the Neumann column (grad_2 = 0) of every image: W - 1, or with a batch of images
    // stacked along columns (rds_create_batch) every img_w-th column; the frame columns
    // left of 0 give negative x.col + e, never an image-last column
    {
        const int iw = a.img_w;
        auto last_col = [&](int c) { return c >= 0 && c < a.W && c % iw == iw - 1; };
        x.right_edge = last_col(x.col + 3);
        x.kx.a = make_float2(last_col(x.col) ? 0.0f : 1.0f, last_col(x.col + 2) ? 0.0f : 1.0f);
        x.kx.b = make_float2(last_col(x.col + 1) ? 0.0f : 1.0f, last_col(x.col + 3) ? 0.0f : 1.0f);
    }
    x.p1i = p1i + x.col;
    x.p2i = p2i + x.col;
    x.vi = vi + x.col;
    x.ci = a.c + x.col;
    // input rows [n, n_last]; the cone reaches S+1 rows up and S rows down, the delay
    // buffer adds one row of latency.  The step count is made even (one extra warm-up
    // row) for the two-state unrolled loop.
    x.n_last = x.Rend - 1 + S + Split<S>::NS;
    int n = x.R0 - (S + 1);
    const bool pro = PRO && !WAVE && x.n_last < a.H - 1;
    if (pro) {  // the prologue's fixed start; one extra step at the end when the count is odd
        n = x.R0 - S - 2;
        if (((x.n_last - n + 1) & 1) != 0) ++x.n_last;
    }
    if (((x.n_last - n + 1) & 1) != 0) --n;
    if (WAVE) wave_need(x, wv, min(n + RING - 1, x.n_last));
#pragma unroll
    for (int r = 0; r < RING; ++r) {
        if (n + r <= x.n_last) stage_row(x, n + r);
        cp_async_commit();
    }
    // the Neumann row H-1 matters whenever the march (cone included) reaches it
    if (x.n_last >= a.H - 1)
        march<S, MODE, ALIGNED, true, WAVE>(x, n, acc_u, acc_v, wv);
    else if (PRO && pro)
        march<S, MODE, ALIGNED, false, WAVE, true>(x, n, acc_u, acc_v, wv);
    else
        march<S, MODE, ALIGNED, false, WAVE>(x, n, acc_u, acc_v, wv);
    cp_async_wait<0>();
    __syncwarp();
}

// Two CTAs (8 warps) per SM: shared memory (94 KB per CTA) and registers both allow 2.
template <int S>
struct MinBlocks {
    static constexpr int value = 2;
};

// PRO: the prologue form (warm-up stages elided, Act), instantiated for MODE_PLAIN and chosen
// per image size at launch
template <int KF, int S, int MODE, bool ALIGNED, bool PRO = false>
__global__ void __launch_bounds__(STENCIL_WARPS * 32, MinBlocks<S>::value)
    k_stencil(const StencilArgs a) {
    static_assert(S >= 1 && S <= KF && KF + 3 <= PAD_R, "stage count");
    static_assert(RING + KF + 3 <= CR, "c ring too short for the stage lags");
    extern __shared__ float4 smem[];  // [warps][RING][3][32] then [warps][CRW]
    // launched as a programmatic dependent of the previous stencil launch: nothing below may
    // run before that grid has completed (its planes, the stop flag)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // tolerance mode: once the stopping rule has fired, the remaining launches are no-ops
    if (a.stop != nullptr && *(volatile const int32_t *)&a.stop->flag != 0) return;
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
    x.chk_r0 = a.chk_r0;
    x.chk_r1 = a.chk_r1;
    x.ring = smem + warp * RING * 96 + lane;
    x.cring = smem + STENCIL_WARPS * RING * 96 + warp * CRW + lane;
    // persistent warps: fetch items from this launch's queue until it is drained
    Wave wv{};
    for (;;) {
        int it = 0;
        if (lane == 0) it = atomicAdd(a.queue, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= n_items) break;  // warp-uniform
        const Item item = a.items[it];
        float acc_u = 0.0f, acc_v = 0.0f;
        run_item<KF, S, MODE, ALIGNED, false, PRO>(x, a, item.strip, item.r0, item.r1, a.p1_in,
                                                   a.p2_in, a.v_in, acc_u, acc_v, wv);
        if (MODE == MODE_CHECK) {  // per-item partial sums, fixed lane order (deterministic)
            double su = acc_u, sv = acc_v;
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                su += __shfl_xor_sync(0xffffffffu, su, off);
                sv += __shfl_xor_sync(0xffffffffu, sv, off);
            }
            if (lane == 0) {
                a.chk[2 * it] = su;
                a.chk[2 * it + 1] = sv;
            }
        }
    }
}


typedef void (*StencilFn)(const StencilArgs);

// Fills t[S][mode][aligned] for S = 1..KF with the kernel instantiations of one k_fuse, and
// pro[S][aligned] with the prologue forms of the plain mode.
template <int KF, int S>
struct Table {
    static void fill(StencilFn (*t)[3][2], StencilFn (*pro)[2]) {
        pro[S][0] = k_stencil<KF, S, MODE_PLAIN, false, true>;
        pro[S][1] = k_stencil<KF, S, MODE_PLAIN, true, true>;
        t[S][0][0] = k_stencil<KF, S, MODE_PLAIN, false>;
        t[S][1][0] = k_stencil<KF, S, MODE_WRITE_U, false>;
        t[S][2][0] = k_stencil<KF, S, MODE_CHECK, false>;
        t[S][0][1] = k_stencil<KF, S, MODE_PLAIN, true>;
        t[S][1][1] = k_stencil<KF, S, MODE_WRITE_U, true>;
        t[S][2][1] = k_stencil<KF, S, MODE_CHECK, true>;
        Table<KF, S - 1>::fill(t, pro);
    }
};
template <int KF>
struct Table<KF, 0> {
    static void fill(StencilFn (*)[3][2], StencilFn (*)[2]) {}
};

constexpr int STENCIL_KF_MAX = 8;
// defined in k_stencil_kf<K>.cu
void stencil_fill_kf1(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf2(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf3(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf4(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf5(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf6(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf7(StencilFn (*t)[3][2], StencilFn (*pro)[2]);
void stencil_fill_kf8(StencilFn (*t)[3][2], StencilFn (*pro)[2]);

}  // namespace rds
