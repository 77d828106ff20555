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

// per RD pixel: neighbour codes, c' and the starting state from the dense planes
__global__ void k_rdc_gather(const RdcSetup a) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int64_t pix = a.list[r];
        const int i = (int)(pix / a.W), j = (int)(pix - (int64_t)i * a.W);
        const bool top = i == 0, bottom = i == a.H - 1, left = j == 0;
        const bool right = j % a.img_w == a.img_w - 1;  // grad_2 = 0 (per image of a batch)
        const int64_t n = a.n;
        a.nbr[0 * n + r] = top ? RDC_BG : a.idxmap[pix - a.W];                 // x - e1
        a.nbr[1 * n + r] = bottom ? RDC_EDGE : a.idxmap[pix + a.W];            // x + e1
        a.nbr[2 * n + r] = left ? RDC_BG : a.idxmap[pix - 1];                  // x - e2
        a.nbr[3 * n + r] = right ? RDC_EDGE : a.idxmap[pix + 1];               // x + e2
        a.nbr[4 * n + r] = (bottom || left) ? RDC_BG : a.idxmap[pix + a.W - 1];  // x + e1 - e2
        a.nbr[5 * n + r] = (top || j == a.W - 1) ? RDC_BG : a.idxmap[pix - a.W + 1];  // x - e1 + e2
        const int64_t o = (int64_t)i * a.pitch + swz(j);
        a.c[r] = a.cplane[o];
        a.p1[r] = a.p1plane[o];
        a.p2[r] = a.p2plane[o];
        a.v[r] = a.vplane[o];
    }
}

// final state back into the dense planes (rho, v swizzled; u, mask natural order)
__global__ void k_rdc_scatter(const RdcSetup a) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.n; r += gridDim.x * blockDim.x) {
        const int64_t pix = a.list[r];
        const int i = (int)(pix / a.W), j = (int)(pix - (int64_t)i * a.W);
        const int64_t o = (int64_t)i * a.pitch + swz(j), on = (int64_t)i * a.pitch + j;
        a.p1plane[o] = a.p1[r];
        a.p2plane[o] = a.p2[r];
        a.vplane[o] = a.v[r];
        const float u = a.u[r];
        a.uplane[on] = u;
        a.mask[on] = u > 0.5f;
    }
}

struct Nb {
    float p1, p2;
};
// rho^k at a neighbour code (0 off RD: rho = 0 on Fg u Bg, Eq. 8); L2 loads, the arrays are
// rewritten by other CTAs between passes
__device__ __forceinline__ Nb rho_at(const float *P1, const float *P2, int code) {
    if (code < 0) return Nb{0.0f, 0.0f};
    return Nb{__ldcg(P1 + code), __ldcg(P2 + code)};
}

// grid-wide barrier k (monotone counter; every CTA adds 1 per barrier)
__device__ __forceinline__ void grid_barrier(unsigned long long *ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1ull);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

}  // namespace

// What a pixel's pass needs besides the state: its neighbour codes and the c' of the pixel
// and of its two forward neighbours (constant over the solve).
struct PixConst {
    int r, up, dn, lf, rt, dl, ur;
    float cx, cd, cr;
};

__device__ __forceinline__ PixConst pix_const(const RdcIter &a, int r) {
    const int64_t n = a.n;
    PixConst q;
    q.r = r;
    q.up = __ldg(a.nbr + r);
    q.dn = __ldg(a.nbr + n + r);
    q.lf = __ldg(a.nbr + 2 * n + r);
    q.rt = __ldg(a.nbr + 3 * n + r);
    q.dl = __ldg(a.nbr + 4 * n + r);
    q.ur = __ldg(a.nbr + 5 * n + r);
    q.cx = __ldg(a.c + r);
    q.cd = q.dn >= 0 ? __ldg(a.c + q.dn) : 0.0f;
    q.cr = q.rt >= 0 ? __ldg(a.c + q.rt) : 0.0f;
    return q;
}

// v^k at y (code, c' of y) from v^{k-1}: Eq. 7 and 9, the pinned u0 off RD; pass 0: v^0
__device__ __forceinline__ float v_of(const float *Vp, int code, float cy, float dy, int k,
                                      float theta) {
    if (code < 0) return code == RDC_FG ? 1.0f : 0.0f;
    const float vp = __ldcg(Vp + code);
    if (k == 0) return vp;
    return __saturatef(__fmaf_rn(cy, -0x1p100f, __fmaf_rn(dy, -theta, vp)));
}

struct PassBufs {
    const float *P1, *P2, *Vp;
    float *Q1, *Q2, *Vo, *U;
};

// pass k at one RD pixel (see the header comment); the same float operations as K3
__device__ __forceinline__ void pix_pass(const PixConst &q, const PassBufs &b, int k, int K,
                                         float tau, float theta, float inv_theta) {
    const Nb px = rho_at(b.P1, b.P2, q.r);
    const Nb pu = rho_at(b.P1, b.P2, q.up), pl = rho_at(b.P1, b.P2, q.lf);
    // div p^k = (p1 - p1(x - e1)) + (p2 - p2(x - e2))
    const float dx = __fadd_rn(__fsub_rn(px.p1, pu.p1), __fsub_rn(px.p2, pl.p2));
    const float vpx = __ldcg(b.Vp + q.r);
    const float ux = __fmaf_rn(dx, -theta, vpx);
    const float vx = k == 0 ? vpx : __saturatef(__fmaf_rn(q.cx, -0x1p100f, ux));
    if (k == K) {  // last pass: u^K and v^K only
        b.Vo[q.r] = vx;
        b.U[q.r] = ux;  // an RD pixel reports u itself (u0 only off RD)
        return;
    }
    const float wx = __fmaf_rn(vx, -inv_theta, dx);
    float g1 = 0.0f, g2 = 0.0f;
    if (q.dn != RDC_EDGE) {  // grad_1 = 0 on row H-1
        const Nb pd = rho_at(b.P1, b.P2, q.dn), pdl = rho_at(b.P1, b.P2, q.dl);
        const float dd = __fadd_rn(__fsub_rn(pd.p1, px.p1), __fsub_rn(pd.p2, pdl.p2));
        g1 = __fsub_rn(__fmaf_rn(v_of(b.Vp, q.dn, q.cd, dd, k, theta), -inv_theta, dd), wx);
    }
    if (q.rt != RDC_EDGE) {  // grad_2 = 0 on an image's last column
        const Nb pr = rho_at(b.P1, b.P2, q.rt), pur = rho_at(b.P1, b.P2, q.ur);
        const float dr = __fadd_rn(__fsub_rn(pr.p1, pur.p1), __fsub_rn(pr.p2, px.p2));
        g2 = __fsub_rn(__fmaf_rn(v_of(b.Vp, q.rt, q.cr, dr, k, theta), -inv_theta, dr), wx);
    }
    const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(q.cx)));
    const float rr = rcp_ax(__fmaf_rn(sqrt_ax(s), tau, 1.0f));
    b.Q1[q.r] = __fmul_rn(__fmaf_rn(g1, tau, px.p1), rr);
    b.Q2[q.r] = __fmul_rn(__fmaf_rn(g2, tau, px.p2), rr);
    if (k > 0) b.Vo[q.r] = vx;
}

__device__ __forceinline__ PassBufs pass_bufs(const RdcIter &a, int k) {
    // selects, not indexing: a runtime index into the parameter arrays costs a stack copy
    const bool odd = k & 1;
    PassBufs b;
    b.P1 = odd ? a.p1[1] : a.p1[0];
    b.P2 = odd ? a.p2[1] : a.p2[0];
    b.Q1 = odd ? a.p1[0] : a.p1[1];
    b.Q2 = odd ? a.p2[0] : a.p2[1];
    b.Vp = (k == 0 || odd) ? a.v[0] : a.v[1];  // v^{k-1} in buffer (k-1)&1; pass 0: v^0
    b.Vo = odd ? a.v[1] : a.v[0];
    b.U = a.u;
    return b;
}

// NPT > 0: every thread owns the fixed pixels t0 + q * stride (q < NPT), whose constants stay
// in registers for the whole solve; NPT = 0: any n, constants reloaded every pass.
template <int NPT>
__global__ void __launch_bounds__(RDC_THREADS) k_rdc_iter(const RdcIter a) {
    const int stride = gridDim.x * blockDim.x;
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    PixConst pc[NPT > 0 ? NPT : 1];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
        const int r = t0 + q * stride;
        pc[q] = r < a.n ? pix_const(a, r) : PixConst{-1};
    }
    for (int k = 0; k <= a.K; ++k) {
        const PassBufs b = pass_bufs(a, k);
        if (NPT > 0) {
#pragma unroll
            for (int q = 0; q < NPT; ++q)
                if (pc[q].r >= 0) pix_pass(pc[q], b, k, a.K, tau, theta, inv_theta);
        } else {
            for (int r = t0; r < a.n; r += stride)
                pix_pass(pix_const(a, r), b, k, a.K, tau, theta, inv_theta);
        }
        if (k < a.K) grid_barrier(a.bar, (unsigned long long)gridDim.x * (unsigned long long)(k + 1));
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
        if (b > 2) b = 2;  // fewer CTAs: a cheaper grid barrier (one atomic per CTA)
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

cudaError_t launch_rdc_scatter(const RdcSetup &a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    int g = (a.n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_rdc_scatter<<<g, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_rdc_iter(const RdcIter &a, int n_sm, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    // the smallest register-resident variant that covers n, else the general one
    RdcFn fn = nullptr;
    int g = 0;
    const int64_t n = a.n;
    if (n <= (int64_t)grid_of<1>(n_sm) * RDC_THREADS) {
        fn = k_rdc_iter<1>;
        g = grid_of<1>(n_sm);
    } else if (n <= (int64_t)grid_of<2>(n_sm) * RDC_THREADS * 2) {
        fn = k_rdc_iter<2>;
        g = grid_of<2>(n_sm);
    } else if (n <= (int64_t)grid_of<4>(n_sm) * RDC_THREADS * 4) {
        fn = k_rdc_iter<4>;
        g = grid_of<4>(n_sm);
    } else if (n <= (int64_t)grid_of<8>(n_sm) * RDC_THREADS * 8) {
        fn = k_rdc_iter<8>;
        g = grid_of<8>(n_sm);
    } else {
        fn = k_rdc_iter<0>;
        g = grid_of<0>(n_sm);
    }
    const int64_t need = (n + RDC_THREADS - 1) / RDC_THREADS;
    if (g > need) g = (int)need;
    void *args[] = {const_cast<RdcIter *>(&a)};
    cudaError_t e = cudaMemsetAsync(a.bar, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel((const void *)fn, dim3(g), dim3(RDC_THREADS), args, 0, s);
}

}  // namespace rds
