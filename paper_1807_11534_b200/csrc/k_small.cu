// k_small.cu -- small images (the paper's own 128 x 128 size) as ONE resident
// thread-block cluster: the whole K-loop of a fixed-K solve in one launch, the state in
// registers, one cluster barrier per iteration (DESIGN.md §5 "resident cluster").
//
// The image is cut into G <= 16 horizontal slabs of R rows (R a compile-time 4, 8 or 16), one
// CTA each; a thread owns ONE column of its slab and keeps that column's state in registers:
// rho1, rho2, v and c' for local rows -2 .. R (the halo rows -2, -1 above and R below come from
// the neighbour slabs).  Iteration k (Eq. 7-9, the rho fixed point of
// PAPER.md:138-141), every row of the column independent of the others (instruction-level
// parallelism R):
//   A  w = div rho - v / theta             rows -1 .. R  (rho2 of the column to the left by shuffle)
//   B  rho' = (rho + tau grad w) rr        rows -1 .. R-1 (w of the column to the right by shuffle;
//                                           rr = 1 / (1 + tau |grad w|), 0 off RD through |c'|)
//   C  u = v - theta div rho', v' = sat(u - c)  rows 0 .. R-1 (rho2' to the left by shuffle)
//   D  the slab's row 0 and rows R-2, R-1 of the new state go into the neighbour CTAs' halo
//      slots (st.shared::cluster), one cluster barrier, the halo rows are read back.
// Warp-edge columns exchange through shared memory (two CTA barriers per iteration).  Every
// float operation is the one k_stencil performs, in the same order (explicit _rn intrinsics,
// MUFU sqrt / rcp, the |c'| and FFMA.SAT folds): the result equals the stencil's bit for bit.
// Rows of the last slab past H - 1, the halo rows beyond the image and the lanes past the last
// column hold the pinned background (rho = 0, v = 0, c' = +inf), which the update keeps.
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

__device__ __forceinline__ unsigned cta_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store a float into the same shared-memory offset of CTA `rank` of the cluster
__device__ __forceinline__ void st_remote(float *local_addr, unsigned rank, float v) {
    unsigned a = (unsigned)__cvta_generic_to_shared(local_addr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
}

constexpr unsigned FULL = 0xffffffffu;

}  // namespace

// Shared memory (floats): halo slots [2][7][NT] (rho1 of rows -2, -1, R; rho2 of -1, R; v of -1,
// R; by iteration parity, so a fast neighbour's next write cannot overtake this CTA's read)
// written by the neighbour CTAs, then the warp-edge exchange rows [2][NW][R + 3].
// columns (threads) per CTA for R rows: the register arrays grow with R
template <int R>
struct SmallCols {
    static constexpr int value = R <= 4 ? 1024 : R <= 8 ? 512 : 256;
};

template <int R>
__global__ void __launch_bounds__(SmallCols<R>::value, 1) k_small(const SmallArgs a) {
    extern __shared__ float sm[];
    constexpr int NR = R + 3;  // local rows -2 .. R, index i + 2
    const int NT = blockDim.x, NW = NT >> 5;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    float *halo = sm;                    // [2 parities][7][NT]
    float *edge = sm + 14 * NT;          // [2][NW][NR]: lane 31's rho2, lane 0's w
    const unsigned rank = cta_rank(), G = a.G;
    const int r0 = (int)rank * R, H = a.H, W = a.W, j = t;
    const bool col_ok = j < W;
    const bool g2_zero = !col_ok || (j % a.img_w) == a.img_w - 1;
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;

    // the column's state, rows -2 .. R (frame rows / columns: the pinned background)
    float p1[NR], p2[NR], v[NR], c[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int gi = r0 + r - 2;
        float x1 = 0.0f, x2 = 0.0f, xv = 0.0f, xc = INFINITY;
        if (col_ok && gi >= -PAD_R && gi < H + PAD_R) {
            const int64_t o = (int64_t)gi * a.pitch + swz(j);
            x1 = a.p1_in[o];
            x2 = a.p2_in[o];
            xv = a.v_in[o];
            xc = a.c[o];
        }
        p1[r] = x1;
        p2[r] = x2;
        v[r] = xv;
        c[r] = xc;
    }
    const bool empty = a.n_rd != nullptr && *a.n_rd == 0;  // every pixel pinned: nothing moves
    const int K = empty ? 0 : a.K;
    // lane 31's rho2 column for the warp to its right (phase A of the first iteration)
    if (lane == 31) {
#pragma unroll
        for (int r = 1; r < NR; ++r) edge[warp * NR + r] = p2[r];
    }
    cluster_sync();  // every CTA running before the first remote store; edge written

    float u_last[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u_last[r] = 0.0f;
    for (int k = 0; k < K; ++k) {
        // A: w on rows -1 .. R; rho2 of the column to the left.  Lane 0 takes the warp to the
        // left's lane 31: rows -1 .. R-1 from `edge` (its rho2' of the previous iteration's phase
        // B; row -1 recomputed there bit-identically to the neighbour's), row R from the halo
        // slot that the CTA below filled for that column.  The interior rows 1 .. R-1 (r = 3 ..
        // NR-2) need no halo row: they run while the cluster barrier of the previous iteration
        // completes (split arrive / wait), the rows -1, 0 and R after it.
        const float *hp = halo + ((k - 1) & 1) * 7 * NT;
        float w[NR];
        auto w_row = [&](int r) {
            float l2 = __shfl_up_sync(FULL, p2[r], 1);
            if (lane == 0) {
                if (warp == 0)
                    l2 = 0.0f;  // the frame column left of column 0
                else if (r < NR - 1 || k == 0)
                    l2 = edge[(warp - 1) * NR + r];
                else
                    l2 = rank + 1 < G ? hp[4 * NT + t - 1] : 0.0f;
            }
            const float d = __fadd_rn(__fsub_rn(p1[r], p1[r - 1]), __fsub_rn(p2[r], l2));
            w[r] = __fmaf_rn(v[r], -inv_theta, d);
        };
#pragma unroll
        for (int r = 3; r < NR - 1; ++r) w_row(r);
        if (k > 0) {
#ifdef RDS_SMALL_NOCLUSTER
            __syncthreads();
#else
            cluster_wait();
#endif
            if (rank > 0) {  // the halo rows of the new state (pushed in iteration k-1)
                p1[0] = hp[0 * NT + t];
                p1[1] = hp[1 * NT + t];
                p2[1] = hp[3 * NT + t];
                v[1] = hp[5 * NT + t];
            }
            if (rank + 1 < G) {
                p1[NR - 1] = hp[2 * NT + t];
                p2[NR - 1] = hp[4 * NT + t];
                v[NR - 1] = hp[6 * NT + t];
            }
        }
        w_row(1);
        w_row(2);
        w_row(NR - 1);
        // lane 0 publishes its w for the warp to the left
#ifndef RDS_SMALL_NOBAR
        __syncthreads();  // (the previous reads of edge are done)
#endif
        if (lane == 0) {
#pragma unroll
            for (int r = 1; r < NR; ++r) edge[NW * NR + warp * NR + r] = w[r];
        }
#ifndef RDS_SMALL_NOBAR
        __syncthreads();
#endif
        // B: rho' on rows -1 .. R-1
        float n1[NR], n2[NR];
#pragma unroll
        for (int r = 1; r < NR - 1; ++r) {
            float wr = __shfl_down_sync(FULL, w[r], 1);
            if (lane == 31) wr = warp + 1 < NW ? edge[NW * NR + (warp + 1) * NR + r] : 0.0f;
            const int gi = r0 + r - 2;
            const float g1 = gi == H - 1 ? 0.0f : __fsub_rn(w[r + 1], w[r]);
            const float g2 = g2_zero ? 0.0f : __fsub_rn(wr, w[r]);
            const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(c[r])));
            const float rr = rcp_ax(__fmaf_rn(sqrt_ax(s), tau, 1.0f));
            n1[r] = __fmul_rn(__fmaf_rn(g1, tau, p1[r]), rr);
            n2[r] = __fmul_rn(__fmaf_rn(g2, tau, p2[r]), rr);
        }
        // lane 31 publishes its rho2' for the warp to the right (phase C now, phase A next)
#ifndef RDS_SMALL_NOBAR
        __syncthreads();
#endif
        if (lane == 31) {
#pragma unroll
            for (int r = 1; r < NR - 1; ++r) edge[warp * NR + r] = n2[r];
        }
#ifndef RDS_SMALL_NOBAR
        __syncthreads();
#endif
        // C: u, v' on rows 0 .. R-1; the new state of rows -1 .. R-1 replaces the old
#pragma unroll
        for (int r = 2; r < NR - 1; ++r) {
            float l2 = __shfl_up_sync(FULL, n2[r], 1);
            if (lane == 0) l2 = warp > 0 ? edge[(warp - 1) * NR + r] : 0.0f;
            const float dn = __fadd_rn(__fsub_rn(n1[r], n1[r - 1]), __fsub_rn(n2[r], l2));
            const float u = __fmaf_rn(dn, -theta, v[r]);
            u_last[r - 2] = fabsf(c[r]) < INFINITY ? u : v[r];
            v[r] = __saturatef(__fmaf_rn(c[r], -0x1p100f, u));
        }
#pragma unroll
        for (int r = 2; r < NR - 1; ++r) {
            p1[r] = n1[r];
            p2[r] = n2[r];
        }
        // D: the new boundary rows into the neighbours' halo slots; then the halo rows back
        float *hs = halo + (k & 1) * 7 * NT;
#ifndef RDS_SMALL_NOPUSH  // (timing experiments only: the RDS_SMALL_NO* variants are wrong)
        if (k + 1 < K) {
            if (rank > 0) {  // my row 0 -> row R of the CTA above
                st_remote(hs + 2 * NT + t, rank - 1, p1[2]);
                st_remote(hs + 4 * NT + t, rank - 1, p2[2]);
                st_remote(hs + 6 * NT + t, rank - 1, v[2]);
            }
            if (rank + 1 < G) {  // my rows R-2 (rho1), R-1 -> rows -2, -1 of the CTA below
                st_remote(hs + 0 * NT + t, rank + 1, p1[R]);
                st_remote(hs + 1 * NT + t, rank + 1, p1[R + 1]);
                st_remote(hs + 3 * NT + t, rank + 1, p2[R + 1]);
                st_remote(hs + 5 * NT + t, rank + 1, v[R + 1]);
            }
        }
#endif
        // arrive now (the pushes released), wait at the next iteration's phase A
#ifndef RDS_SMALL_NOCLUSTER
        if (k + 1 < K) cluster_arrive();
#endif
    }
    // outputs: u and the mask of the last iteration (u0 = v when nothing moved), the state
    if (!col_ok) return;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int gi = r0 + r;
        if (gi >= H) break;
        const int64_t o = (int64_t)gi * a.pitch;
        const float ou = K > 0 ? u_last[r] : v[r + 2];
        a.u_out[o + j] = ou;
        a.mask_out[o + j] = ou > 0.5f;
        if (K > 0) {
            a.p1_out[o + swz(j)] = p1[r + 2];
            a.p2_out[o + swz(j)] = p2[r + 2];
            a.v_out[o + swz(j)] = v[r + 2];
        }
    }
}

static int small_threads(int W) { return (W + 31) / 32 * 32; }
static size_t small_smem(int R, int W) {
    const int NT = small_threads(W);
    return sizeof(float) * (size_t)(14 * NT + 2 * (NT / 32) * (R + 3));
}

// Slabs for an H x W image: R in {4, 8, 16} (the smallest with G = ceil(H / R) <= 16 CTAs),
// one thread per column (W <= 1024 / 512 / 256 for R = 4 / 8 / 16).  false if the image does
// not fit one cluster.
bool small_plan(int64_t H, int64_t W, int *G_out, int *R_out) {
    if (H < 1 || W < 1) return false;
    for (int R : {4, 8, 16}) {
        const int64_t G = (H + R - 1) / R;
        const int cols = R <= 4 ? SmallCols<4>::value : R <= 8 ? SmallCols<8>::value
                                                               : SmallCols<16>::value;
        if (G <= SMALL_MAX_CTAS && W <= cols) {
            *G_out = (int)G;
            *R_out = R;
            return true;
        }
    }
    return false;
}

typedef void (*SmallFn)(const SmallArgs);
static SmallFn small_fn(int R) {
    return R == 4 ? k_small<4> : R == 8 ? k_small<8> : R == 16 ? k_small<16> : nullptr;
}

static cudaLaunchConfig_t small_cfg(const SmallArgs &a, cudaLaunchAttribute *attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.G);
    cfg.blockDim = dim3(small_threads(a.W));
    cfg.dynamicSmemBytes = small_smem(a.R, a.W);
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

static cudaError_t small_prepare(SmallFn fn, const SmallArgs &a) {
    cudaError_t e = cudaFuncSetAttribute((const void *)fn,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)small_smem(a.R, a.W));
    if (e == cudaSuccess && a.G > 8)
        e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                 1);
    return e;
}

cudaError_t launch_small(const SmallArgs &a, cudaStream_t s) {
    SmallFn fn = small_fn(a.R);
    if (!fn) return cudaErrorInvalidValue;
    cudaError_t e = small_prepare(fn, a);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = small_cfg(a, attr);
    cfg.stream = s;
    void *args[] = {const_cast<SmallArgs *>(&a)};
    return cudaLaunchKernelExC(&cfg, (const void *)fn, args);
}

// Can one cluster of G CTAs of this shape be scheduled here?
bool small_cluster_fits(const SmallArgs &a) {
    SmallFn fn = small_fn(a.R);
    if (!fn || small_prepare(fn, a) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = small_cfg(a, attr);
    int n = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&n, (const void *)fn, &cfg) == cudaSuccess &&
                    n >= 1;
    (void)cudaGetLastError();
    return ok;
}

}  // namespace rds
