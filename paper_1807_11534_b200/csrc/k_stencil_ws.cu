// k_stencil_ws.cu -- K3 with warp-specialised stage chains (RDS_OPT_WS).
//
// The same S-stage software pipeline as k_stencil (k_stencil_impl.cuh: the same stage(), the
// same float operations in the same order, so the results are bit-identical), but the chains
// of stages that k_stencil joins through one-row delay buffers inside ONE warp are run by
// DIFFERENT warps of a CTA: warp C owns stages [sp(C), sp(C+1)) of a work item, and the row a
// chain emits in row step n reaches the next chain's warp through a shared-memory hand-off
// slot in row step n + 1 -- exactly the one-row delay of k_stencil's split, so the row lags
// (and everything computed) are unchanged.  Each warp then holds the state of 2-3 stages
// instead of S, so 3-5 CTAs fit an SM instead of two 4-warp CTAs: 4-5 independent instruction
// streams per SM sub-partition instead of 2 to overlap the MUFU, FMA and issue pipes the
// stencil is co-bound on (DESIGN.md §5 "what binds").
//
// Per row step n of an item, warp C:
//   C = 0   : takes input row n (rho1, rho2, v) from its cp.async ring and forms div rho there;
//   C > 0   : takes chain C-1's emission of row step n-1 (rho1, rho2, v, div rho) from slot
//             (C-1, (n-1) & 1) of the hand-off buffer;
//   runs its stages;
//   C < NC-1: writes its emission to slot (C, n & 1); the last chain stores the level-S row;
//   C = 0   : refills the ring with row n + RING (rho1, rho2, v and c');
//   then one CTA barrier: after it, the slots written in step n and the c' rows warp 0 waited
//   for are visible to every warp, and the slots read in step n may be overwritten.
// The c' ring is shared by the CTA (every stage reads c' at its own lagging row).
#include <stdlib.h>

#include "k_stencil_impl.cuh"

namespace rds {

// NC chains of near-equal stage counts; lag(t) = chain boundaries <= t (the row delay)
template <int S, int NC>
struct SplitWS {
    static constexpr int NS = NC - 1;
    __host__ __device__ static constexpr int sp(int k) { return (k * S) / NC; }
    __host__ __device__ static constexpr int lag(int t) {
        int n = 0;
        for (int k = 1; k <= NS; ++k) n += sp(k) <= t;
        return n;
    }
};

__device__ __forceinline__ void ws_st_pred(float *p, const Q &x, bool pr) {  // swizzled
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n"
        " @p st.global.v4.f32 [%1], {%2, %3, %4, %5};\n}\n" ::"r"((int)pr),
        "l"(p), "f"(x.a.x), "f"(x.a.y), "f"(x.b.x), "f"(x.b.y)
        : "memory");
}

constexpr int WS_HAND = 4 * 32;  // float4 per hand-off slot: rho1, rho2, v, div rho x 32 lanes
// shared memory in float4: rho/v ring (warp 0), c' ring (doubled), hand-off slots, item word
__host__ __device__ constexpr int ws_smem_f4(int nc) {
    return RING * 96 + 2 * CR * 32 + (nc - 1) * 2 * WS_HAND;
}
__host__ __device__ constexpr int ws_smem_bytes(int nc) { return (ws_smem_f4(nc) + 1) * 16; }

#ifndef RDS_WS_MINB
#define RDS_WS_MINB 0
#endif

template <int N>
struct WsState {
    Q p1[N], p2[N], v[N], w[N];
    Q q1;  // rho1 the chain's last stage emitted in the previous row step
};

__device__ __forceinline__ void bar_rows(int nthreads) {  // named barrier 1: the row steps
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int S, int NC, int C, bool LAST>
__device__ __forceinline__ void ws_step(const WsState<SplitWS<S, NC>::sp(C + 1) - SplitWS<S, NC>::sp(C)> &A,
                                        WsState<SplitWS<S, NC>::sp(C + 1) - SplitWS<S, NC>::sp(C)> &B,
                                        int n, const Ctx &x, const float4 *hin, float4 *hout) {
    using SP = SplitWS<S, NC>;
    constexpr int T0 = SP::sp(C), T1 = SP::sp(C + 1), N = T1 - T0;
    Q in1, in2, inv, ind;
    if (C == 0) {
        cp_async_wait<RING - 1>();
        const float4 *slot = x.ring + (n & (RING - 1)) * 96;
        in1 = ldq(slot[0]);
        in2 = ldq(slot[32]);
        inv = ldq(slot[64]);
        ind = div_q(in1, A.p1[0], in2);  // div rho of level 0 at row n
    } else {
        const float4 *h = hin + ((n - 1) & 1) * WS_HAND;
        in1 = ldq(h[0]);
        in2 = ldq(h[32]);
        inv = ldq(h[64]);
        ind = ldq(h[96]);
    }
    const float4 *crow = x.cring + ((n & (CR - 1)) + CR) * 32;  // row n; row n-L at -32 L
    Q uu;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const int t = T0 + i;
        const int m = n - t - 1 - SP::lag(t);  // row emitted (level t+1)
        const Q &q1 = (i == N - 1) ? A.q1 : A.p1[(i + 1 < N) ? i + 1 : 0];
        const float4 c4 = crow[-32 * (n - m)];
        Q o1, o2, ov, od;
        stage<false, true, LAST>(A.p1[i], A.p2[i], A.v[i], A.w[i], q1, in1, in2, inv, ind, c4, m,
                                 x, B.p1[i], B.p2[i], B.v[i], B.w[i], o1, o2, ov, od, uu);
        in1 = o1;
        in2 = o2;
        inv = ov;
        ind = od;
    }
    B.q1 = in1;
    if (C < NC - 1) {
        float4 *h = hout + (n & 1) * WS_HAND;
        stq(reinterpret_cast<float *>(h), in1);
        stq(reinterpret_cast<float *>(h + 32), in2);
        stq(reinterpret_cast<float *>(h + 64), inv);
        stq(reinterpret_cast<float *>(h + 96), ind);
    } else {
        const int m = n - S - SP::NS;  // the level-S row of this step
        const bool st = x.store_lane && m >= x.R0 && m < x.Rend;
        const int64_t o = (int64_t)m * x.pitch + x.col;
        ws_st_pred(x.p1o + o, in1, st);
        ws_st_pred(x.p2o + o, in2, st);
        ws_st_pred(x.vo + o, inv, st);
    }
    if (C == 0) {
        if (n + RING <= x.n_last) stage_row(x, n + RING);
        cp_async_commit();
    }
    bar_rows(NC * 32);
}

template <int S, int NC, int C, bool LAST>
__device__ __forceinline__ void ws_march(const Ctx &x, int n, const float4 *hin, float4 *hout) {
    using SP = SplitWS<S, NC>;
    constexpr int N = SP::sp(C + 1) - SP::sp(C);
    WsState<N> A, B;
#pragma unroll
    for (int i = 0; i < N; ++i) A.p1[i] = A.p2[i] = A.v[i] = A.w[i] = zeroq();
    A.q1 = zeroq();
    for (; n <= x.n_last; n += 2) {
        ws_step<S, NC, C, LAST>(A, B, n, x, hin, hout);
        ws_step<S, NC, C, LAST>(B, A, n + 1, x, hin, hout);
    }
}

template <int S, int NC, int C>
__device__ __forceinline__ void ws_chain(const Ctx &x, int n, bool last, float4 *hand) {
    const int lane = threadIdx.x & 31;
    const float4 *hin = hand + (C > 0 ? C - 1 : 0) * 2 * WS_HAND + lane;
    float4 *hout = hand + (C < NC - 1 ? C : 0) * 2 * WS_HAND + lane;
    if (last)
        ws_march<S, NC, C, true>(x, n, hin, hout);
    else
        ws_march<S, NC, C, false>(x, n, hin, hout);
}

template <int S, int NC, int C = 0>
struct WsDispatch {
    __device__ static __forceinline__ void run(int warp, const Ctx &x, int n, bool last,
                                               float4 *hand) {
        if (warp == C)
            ws_chain<S, NC, C>(x, n, last, hand);
        else
            WsDispatch<S, NC, C + 1>::run(warp, x, n, last, hand);
    }
};
template <int S, int NC>
struct WsDispatch<S, NC, NC> {
    __device__ static __forceinline__ void run(int, const Ctx &, int, bool, float4 *) {}
};

template <int S, int NC>
__global__ void __launch_bounds__(NC * 32, RDS_WS_MINB) k_stencil_ws(const StencilArgs a) {
    static_assert(S >= NC && NC >= 2, "at least one stage per chain");
    static_assert(RING + S + NC <= CR, "c ring too short for the stage lags");
    extern __shared__ float4 smem[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.stop != nullptr && *(volatile const int32_t *)&a.stop->flag != 0) return;
    using SP = SplitWS<S, NC>;
    constexpr int WV = wv_of(S), LH = lh_of(S);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int *item_word = reinterpret_cast<int *>(smem + ws_smem_f4(NC));
    float4 *hand = smem + RING * 96 + 2 * CR * 32;
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
    x.ring = smem + lane;
    x.cring = smem + RING * 96 + lane;
    const int n_items = *a.n_items;
    for (;;) {
        __syncthreads();  // every warp is done with the previous item (rings, slots)
        if (threadIdx.x == 0) *item_word = atomicAdd(a.queue, 1);
        __syncthreads();
        const int it = *item_word;
        if (it >= n_items) break;  // CTA-uniform
        const Item item = a.items[it];
        // lane geometry of the item's strip (as run_item)
        x.R0 = item.r0;
        x.Rend = item.r1;
        x.col = item.strip * WV - LH + 4 * lane;
        x.store_lane = (4 * lane >= LH) && (4 * lane < LH + WV);
        {
            const int iw = a.img_w;
            auto last_col = [&](int c) { return c >= 0 && c < a.W && c % iw == iw - 1; };
            x.right_edge = last_col(x.col + 3);
            x.kx.a = make_float2(1.0f, 1.0f);  // (ALIGNED: the packed edge uses right_edge)
            x.kx.b = make_float2(1.0f, 1.0f);
        }
        x.p1i = a.p1_in + x.col;
        x.p2i = a.p2_in + x.col;
        x.vi = a.v_in + x.col;
        x.ci = a.c + x.col;
        x.n_last = x.Rend - 1 + S + SP::NS;
        int n = x.R0 - (S + 1);
        if (((x.n_last - n + 1) & 1) != 0) --n;
        if (warp == 0) {
#pragma unroll
            for (int r = 0; r < RING; ++r) {
                if (n + r <= x.n_last) stage_row(x, n + r);
                cp_async_commit();
            }
        }
        WsDispatch<S, NC>::run(warp, x, n, x.n_last >= a.H - 1, hand);
        if (warp == 0) cp_async_wait<0>();
    }
}

// ---------------------------------------------------------------------------------------
// dispatch: (S, NC) instantiations; RDS_WS_LIST overrides for experiments
// ---------------------------------------------------------------------------------------
#ifndef RDS_WS_LIST
#define RDS_WS_LIST(X) X(6, 3) X(7, 3) X(8, 4)
#endif

typedef void (*WsFn)(const StencilArgs);
struct WsEntry {
    WsFn fn;
    int nc;
};

static WsEntry ws_lookup(int s) {
    static WsEntry table[STENCIL_KF_MAX + 4] = {};
    static bool init = false;
    if (!init) {
#define RDS_WS_FILL(S_, NC_)                                                           \
    if (S_ < (int)(sizeof table / sizeof table[0])) {                                  \
        table[S_] = WsEntry{k_stencil_ws<S_, NC_>, NC_};                               \
        cudaFuncSetAttribute((const void *)k_stencil_ws<S_, NC_>,                      \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, ws_smem_bytes(NC_)); \
    }
        RDS_WS_LIST(RDS_WS_FILL)
#undef RDS_WS_FILL
        init = true;
    }
    if (s < 0 || s >= (int)(sizeof table / sizeof table[0])) return WsEntry{nullptr, 0};
    return table[s];
}

bool ws_available(int stages) { return ws_lookup(stages).fn != nullptr; }

int ws_blocks_per_sm(int stages) {
    const WsEntry e = ws_lookup(stages);
    if (!e.fn) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, e.fn, e.nc * 32,
                                                      ws_smem_bytes(e.nc)) != cudaSuccess)
        return 0;
    return nb;
}

cudaError_t launch_stencil_ws(int stages, const StencilArgs &a, int grid, cudaStream_t s) {
    const WsEntry e = ws_lookup(stages);
    if (!e.fn) return cudaErrorInvalidValue;
    if (grid <= 0) return cudaSuccess;
    static const bool pdl = getenv("RDS_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(e.nc * 32);
    cfg.dynamicSmemBytes = ws_smem_bytes(e.nc);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void *args[] = {const_cast<StencilArgs *>(&a)};
    cudaLaunchKernelExC(&cfg, (const void *)e.fn, args);
    return cudaGetLastError();
}

}  // namespace rds
