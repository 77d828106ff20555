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
// clamp(u - c, 0, 1) reproduces the pinned u0 exactly and "RD" is |c| < inf.
//
// Execution model.  Each warp owns one work item: a strip of 128 columns
// (4 per lane, float4 loads/stores, 512 B per row per array) of which WV = wv_of(KF) are
// output columns, marching down the rows of a chunk.  The S iterations are a software
// pipeline in registers: stage t consumes level t-1 at row m+1 and emits level t at row m,
// so each input row is read once from HBM and each output row written once per S
// iterations.  Horizontal neighbours come from warp shuffles (3 per stage per row); the
// dependency cone (KF+1 columns/rows behind, KF ahead) is recomputed redundantly at the
// strip and chunk edges instead of being exchanged.  Stage state per pixel: rho1, rho2, v,
// c, w of level t-1 at row m and rho1 of level t at row m-1.
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
__device__ __forceinline__ float4 ldg4(const float *p) {
    return __ldg(reinterpret_cast<const float4 *>(p));
}
__device__ __forceinline__ void st4(float *p, const float (&x)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(x[0], x[1], x[2], x[3]);
}

template <int KF, int S, bool WRITE_U>
__global__ void __launch_bounds__(STENCIL_WARPS * 32) k_stencil(const StencilArgs a) {
    static_assert(S >= 1 && S <= KF && KF + 1 <= PAD_R, "stage count");
    constexpr int LH = lh_of(KF), WV = wv_of(KF);
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int widx = blockIdx.x * STENCIL_WARPS + (threadIdx.x >> 5);
    if (widx >= *a.n_items) return;  // warp-uniform exit
    const int item = a.items[widx];
    const int b = item / a.n_strips, s = item - b * a.n_strips;
    const int R0 = b * a.rows;
    const int Rend = min(R0 + a.rows, a.H);
    const int col = s * WV - LH + 4 * lane;
    const bool store_lane = (4 * lane >= LH) && (4 * lane < LH + WV);
    const int64_t pitch = a.pitch;
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    float kx[4];  // grad_2 = 0 on column W-1 (Neumann)
#pragma unroll
    for (int e = 0; e < 4; ++e) kx[e] = (col + e == a.W - 1) ? 0.0f : 1.0f;

    const float *p1i = a.p1_in + col, *p2i = a.p2_in + col, *vi = a.v_in + col,
                *ci = a.c + col;

    float pa1[S][4], pa2[S][4], va[S][4], ca[S][4], wa[S][4], q1[S][4];
#pragma unroll
    for (int t = 0; t < S; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e)
            pa1[t][e] = pa2[t][e] = va[t][e] = ca[t][e] = wa[t][e] = q1[t][e] = 0.0f;

    int n = R0 - (S + 1);             // first input row (cone reaches S+1 rows up)
    const int n_last = Rend - 1 + S;  // last input row (cone reaches S rows down)
    int64_t off = (int64_t)n * pitch;
    float4 x1 = ldg4(p1i + off), x2 = ldg4(p2i + off), xv = ldg4(vi + off),
           xc = ldg4(ci + off);
    for (; n <= n_last; ++n) {
        float in1[4] = {x1.x, x1.y, x1.z, x1.w};
        float in2[4] = {x2.x, x2.y, x2.z, x2.w};
        float inv[4] = {xv.x, xv.y, xv.z, xv.w};
        float inc[4] = {xc.x, xc.y, xc.z, xc.w};
        if (n < n_last) {  // prefetch the next input row
            off += pitch;
            x1 = ldg4(p1i + off);
            x2 = ldg4(p2i + off);
            xv = ldg4(vi + off);
            xc = ldg4(ci + off);
        }
#pragma unroll
        for (int t = 0; t < S; ++t) {
            const int m = n - t - 1;  // row emitted by this stage (level t+1)
            // w at row m+1, level t
            const float l2 = __shfl_up_sync(FULL, in2[3], 1);
            float w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float p2l = e ? in2[e - 1] : l2;
                w[e] = in1[e] - pa1[t][e] + in2[e] - p2l - inv[e] * inv_theta;
            }
            // rho-step at row m
            const float wr = __shfl_down_sync(FULL, wa[t][0], 1);
            const bool last_row = (m == a.H - 1);
            float np1[4], np2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float g1 = last_row ? 0.0f : (w[e] - wa[t][e]);
                const float g2 = ((e < 3 ? wa[t][e + 1] : wr) - wa[t][e]) * kx[e];
                const float rr = rcp_approx(1.0f + tau * sqrt_approx(g1 * g1 + g2 * g2));
                const bool rd = fabsf(ca[t][e]) < INFINITY;
                np1[e] = rd ? (pa1[t][e] + tau * g1) * rr : 0.0f;
                np2[e] = rd ? (pa2[t][e] + tau * g2) * rr : 0.0f;
            }
            // u-step and v-step at row m
            const float l2n = __shfl_up_sync(FULL, np2[3], 1);
            float nv[4], uu[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float d = np1[e] - q1[t][e] + np2[e] - (e ? np2[e - 1] : l2n);
                const float u = va[t][e] - theta * d;
                nv[e] = fminf(fmaxf(u - ca[t][e], 0.0f), 1.0f);
                uu[e] = (fabsf(ca[t][e]) < INFINITY) ? u : va[t][e];
            }
            float oc[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                oc[e] = ca[t][e];
                q1[t][e] = np1[e];
                pa1[t][e] = in1[e];
                pa2[t][e] = in2[e];
                va[t][e] = inv[e];
                ca[t][e] = inc[e];
                wa[t][e] = w[e];
                in1[e] = np1[e];
                in2[e] = np2[e];
                inv[e] = nv[e];
                inc[e] = oc[e];
            }
            if (t == S - 1) {
                if (store_lane && m >= R0 && m < Rend) {
                    const int64_t o = (int64_t)m * pitch + col;
                    st4(a.p1_out + o, np1);
                    st4(a.p2_out + o, np2);
                    st4(a.v_out + o, nv);
                    if (WRITE_U) {
                        st4(a.u_out + o, uu);
                        *reinterpret_cast<uchar4 *>(a.mask_out + o) =
                            make_uchar4(uu[0] > 0.5f, uu[1] > 0.5f, uu[2] > 0.5f,
                                        uu[3] > 0.5f);
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// dispatch over (KF, S, WRITE_U)
// ---------------------------------------------------------------------------------------
typedef void (*StencilFn)(const StencilArgs);

template <int KF, int S>
struct Table {
    static void fill(StencilFn (*t)[2]) {
        t[S][0] = k_stencil<KF, S, false>;
        t[S][1] = k_stencil<KF, S, true>;
        Table<KF, S - 1>::fill(t);
    }
};
template <int KF>
struct Table<KF, 0> {
    static void fill(StencilFn (*)[2]) {}
};

#define RDS_KF_LIST(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)

static const int kKfMax = 8;

static StencilFn lookup(int kf, int stages, bool write_u) {
    static StencilFn table[kKfMax + 1][kKfMax + 1][2];
    static bool init = false;
    if (!init) {
#define RDS_FILL(K) Table<K, K>::fill(table[K]);
        RDS_KF_LIST(RDS_FILL)
#undef RDS_FILL
        init = true;
    }
    if (kf < 1 || kf > kKfMax || stages < 1 || stages > kf) return nullptr;
    return table[kf][stages][write_u ? 1 : 0];
}

bool kf_supported(int kf) { return lookup(kf, 1, false) != nullptr; }

int kf_list(int32_t *out, int cap) {
    int n = 0;
    for (int k = 1; k <= kKfMax; ++k)
        if (kf_supported(k)) {
            if (n < cap && out) out[n] = k;
            ++n;
        }
    return n;
}

cudaError_t launch_stencil(int kf, int stages, bool write_u, const StencilArgs &a, int grid,
                           cudaStream_t s) {
    StencilFn fn = lookup(kf, stages, write_u);
    if (!fn) return cudaErrorInvalidValue;
    if (grid <= 0) return cudaSuccess;
    fn<<<grid, STENCIL_WARPS * 32, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace rds
