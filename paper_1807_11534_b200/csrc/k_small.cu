// k_small.cu -- small images (the paper's own 128 x 128 size) as ONE resident
// thread-block cluster: the whole K-loop of a fixed-K solve in one launch, the state in
// shared memory, one cluster barrier per iteration (DESIGN.md §5 "resident cluster").
//
// The image is cut into G horizontal slabs of R rows, one CTA each (G <= 16, one cluster).  A
// CTA keeps its slab's state (rho1, rho2, v, ping-pong) plus halo rows in shared memory:
// rows -2, -1 above (rho1 of -2; rho1, rho2, v of -1) and row R below, and one frame column on
// each side.  Iteration k (Eq. 7-9, the rho fixed point of PAPER.md:138-141):
//   A  w = div rho - v / theta             on rows -1 .. R   (own rows and the two halo rows)
//   B  rho' = (rho + tau grad w) rr        on rows -1 .. R-1 (rr = 1 / (1 + tau |grad w|); 0 off
//                                           RD through |c'|; row -1 recomputed locally)
//   C  u = v - theta div rho', v' = sat(u - c)  on the own rows
//   D  the slab's first row and last two rows of the new state are pushed into the neighbour
//      CTAs' halo rows (st.shared::cluster), then one cluster barrier (release / acquire).
// The halo rows let every CTA compute the rho' of the row above its slab itself, so one
// barrier per iteration suffices.  Every float operation is the one k_stencil performs, in the
// same order (explicit _rn intrinsics, MUFU sqrt / rcp, the |c'| and FFMA.SAT folds), so the
// result equals the dense path's bit for bit.  Rows of the last slab past H - 1 and the frame
// columns hold the pinned background (rho = 0, v = 0, c' = +inf) and stay so.
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
// store a float into the same shared-memory offset of CTA `rank` of the cluster
__device__ __forceinline__ void st_remote(float *local_addr, unsigned rank, float v) {
    unsigned a = (unsigned)__cvta_generic_to_shared(local_addr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(ra), "f"(v) : "memory");
}

}  // namespace

// Shared-memory layout of one CTA (floats): planes of RH = R + 3 rows (local rows -2 .. R) by
// WP = W + 2 columns (local columns -1 .. W); element (i, j) at (i + 2) * WP + j + 1.
struct SmallGeom {
    int R, WP, RH;
    __host__ __device__ int plane() const { return RH * WP; }
    // P1[2], P2[2], V[2], C, Wt, then one row: rho1' of local row -1 (phase B, local use),
    // then W bytes of image-last-column flags
    __host__ __device__ int floats() const { return 8 * plane() + WP + (WP + 3) / 4; }
};

__global__ void __launch_bounds__(SMALL_THREADS, 1) k_small(const SmallArgs a) {
    extern __shared__ float sm[];
    const SmallGeom g{a.R, a.W + 2, a.R + 3};
    const int P = g.plane();
    // ping-pong planes at sm + b*P (rho1), sm + (2+b)*P (rho2), sm + (4+b)*P (v); then c', w,
    // the scratch row rho1' of local row -1, and per column whether it is an image's last
    float *C = sm + 6 * P, *Wt = sm + 7 * P, *Qm = sm + 8 * P;
    uint8_t *lastc = reinterpret_cast<uint8_t *>(Qm + g.WP);
    const unsigned rank = cta_rank(), G = a.G;
    const int r0 = (int)rank * a.R;              // first global row of the slab
    const int W = a.W, WP = g.WP, H = a.H;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 columns x 16 rows per pass
    constexpr int TY = SMALL_THREADS / 32;
    auto at = [&](int i, int j) { return (i + 2) * WP + j + 1; };
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;

    // an empty band: every pixel is pinned, so u = u0 and the state does not move
    const bool empty = a.n_rd != nullptr && *a.n_rd == 0;

    // load the slab with its halo rows / columns from the dense planes (frame rows and
    // columns included: they hold the pinned background) -- both ping-pong copies
    for (int i = ty - 2; i <= a.R; i += TY) {
        const int gi = r0 + i;
        // rows past H inside the padded frame hold the background there; rows further down
        // (a partial last slab taller than the frame) get it here
        const bool in_pad = gi >= -PAD_R && gi < H + PAD_R;
        for (int j = tx - 1; j <= W; j += 32) {
            float p1 = 0.0f, p2 = 0.0f, v = 0.0f, c = INFINITY;
            if (in_pad) {
                const int64_t o = (int64_t)gi * a.pitch + swz(j);
                p1 = a.p1_in[o];
                p2 = a.p2_in[o];
                v = a.v_in[o];
                c = a.c[o];
            }
            const int e = at(i, j);
            sm[e] = sm[P + e] = p1;
            sm[2 * P + e] = sm[3 * P + e] = p2;
            sm[4 * P + e] = sm[5 * P + e] = v;
            C[e] = c;
            Wt[e] = 0.0f;
        }
    }
    for (int j = threadIdx.x; j < WP; j += SMALL_THREADS) Qm[j] = 0.0f;
    for (int j = threadIdx.x; j < W; j += SMALL_THREADS) lastc[j] = (j % a.img_w) == a.img_w - 1;
    cluster_sync();  // every CTA's shared memory initialised before any remote store

    int cur = 0;
    const int K = empty ? 0 : a.K;
    for (int k = 0; k < K; ++k) {
        const float *p1 = sm + cur * P, *p2 = sm + (2 + cur) * P, *v = sm + (4 + cur) * P;
        float *q1 = sm + (cur ^ 1) * P, *q2 = sm + (2 + (cur ^ 1)) * P;
        float *vo = sm + (4 + (cur ^ 1)) * P;
        // A: w on local rows -1 .. R
        for (int i = ty - 1; i <= a.R; i += TY)
            for (int j = tx; j < W; j += 32) {
                const int o = at(i, j);
                const float d =
                    __fadd_rn(__fsub_rn(p1[o], p1[o - WP]), __fsub_rn(p2[o], p2[o - 1]));
                Wt[o] = __fmaf_rn(v[o], -inv_theta, d);
            }
        __syncthreads();
        // B: rho' on local rows -1 .. R-1 (row -1: rho1' only, into the scratch row Qm; the
        // neighbour above pushes its own copy of that row into q* for the next iteration)
        for (int i = ty - 1; i < a.R; i += TY) {
            const bool g1_zero = r0 + i == H - 1;
            for (int j = tx; j < W; j += 32) {
                const int o = at(i, j);
                const float w0 = Wt[o];
                const float g1 = g1_zero ? 0.0f : __fsub_rn(Wt[o + WP], w0);
                const float g2 = lastc[j] ? 0.0f : __fsub_rn(Wt[o + 1], w0);
                const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(C[o])));
                const float rr = rcp_ax(__fmaf_rn(sqrt_ax(s), tau, 1.0f));
                const float n1 = __fmul_rn(__fmaf_rn(g1, tau, p1[o]), rr);
                if (i < 0) {
                    Qm[j + 1] = n1;
                } else {
                    q1[o] = n1;
                    q2[o] = __fmul_rn(__fmaf_rn(g2, tau, p2[o]), rr);
                }
            }
        }
        __syncthreads();
        // C: u, v' on the own rows; the last iteration also writes u and the mask
        const bool last = k == K - 1;
        for (int i = ty; i < a.R; i += TY) {
            const int gi = r0 + i;
            for (int j = tx; j < W; j += 32) {
                const int o = at(i, j);
                const float up = i == 0 ? Qm[j + 1] : q1[o - WP];
                const float dn = __fadd_rn(__fsub_rn(q1[o], up), __fsub_rn(q2[o], q2[o - 1]));
                const float u = __fmaf_rn(dn, -theta, v[o]);
                const float c = C[o];
                vo[o] = __saturatef(__fmaf_rn(c, -0x1p100f, u));
                if (last && gi < H) {
                    const int64_t go = (int64_t)gi * a.pitch + j;
                    const float ou = fabsf(c) < INFINITY ? u : v[o];
                    a.u_out[go] = ou;
                    a.mask_out[go] = ou > 0.5f;
                }
            }
        }
        // D: push the new boundary rows into the neighbours' halo rows (their buffer cur ^ 1);
        // the rows are read back from shared memory, so the CTA must have finished phase C
#ifndef RDS_SMALL_NOPUSH  // (timing experiments only: RDS_SMALL_NOPUSH / _NOCLUSTER are wrong)
        if (k + 1 < K) {
            __syncthreads();
            for (int j = threadIdx.x; j < W; j += SMALL_THREADS) {
                if (rank > 0) {  // my row 0 -> row R of the CTA above
                    const int o = at(0, j), t = at(a.R, j);
                    st_remote(q1 + t, rank - 1, q1[o]);
                    st_remote(q2 + t, rank - 1, q2[o]);
                    st_remote(vo + t, rank - 1, vo[o]);
                }
                if (rank + 1 < G) {  // my rows R-2 (rho1), R-1 -> rows -2, -1 of the CTA below
                    const int o2 = at(a.R - 2, j), o1 = at(a.R - 1, j);
                    st_remote(q1 + at(-2, j), rank + 1, q1[o2]);
                    st_remote(q1 + at(-1, j), rank + 1, q1[o1]);
                    st_remote(q2 + at(-1, j), rank + 1, q2[o1]);
                    st_remote(vo + at(-1, j), rank + 1, vo[o1]);
                }
            }
        }
#endif
#ifdef RDS_SMALL_NOCLUSTER
        __syncthreads();
#else
        cluster_sync();
#endif
        cur ^= 1;
    }
    if (empty) {  // u = u0 (= v, pinned) and the mask; the state stays as loaded
        for (int i = ty; i < a.R; i += TY) {
            const int gi = r0 + i;
            if (gi >= H) continue;
            for (int j = tx; j < W; j += 32) {
                const float ou = sm[4 * P + at(i, j)];
                a.u_out[(int64_t)gi * a.pitch + j] = ou;
                a.mask_out[(int64_t)gi * a.pitch + j] = ou > 0.5f;
            }
        }
        return;
    }
    // final state into the dense ping-pong buffer `out` (swizzled planes)
    const float *p1 = sm + cur * P, *p2 = sm + (2 + cur) * P, *v = sm + (4 + cur) * P;
    for (int i = ty; i < a.R; i += TY) {
        const int gi = r0 + i;
        if (gi >= H) continue;
        for (int j = tx; j < W; j += 32) {
            const int o = at(i, j);
            const int64_t go = (int64_t)gi * a.pitch + swz(j);
            a.p1_out[go] = p1[o];
            a.p2_out[go] = p2[o];
            a.v_out[go] = v[o];
        }
    }
}

// Shared memory bytes of one CTA for R rows of width W; 0 if the layout cannot hold them.
size_t small_smem_bytes(int R, int W) {
    const SmallGeom g{R, W + 2, R + 3};
    return sizeof(float) * (size_t)g.floats();
}

// The cluster (G slabs of R rows) for an H x W image, or G = 0 if the image does not fit one
// cluster's shared memory / rows per slab.
bool small_plan(int64_t H, int64_t W, int *G_out, int *R_out) {
    if (H < 2 || W < 1 || W > 4096) return false;
    for (int G = 1; G <= SMALL_MAX_CTAS; ++G) {
        const int R = (int)((H + G - 1) / G);
        if (R < 2) break;
        if (small_smem_bytes(R, (int)W) <= SMALL_MAX_SMEM) {
            // more CTAs = less work per SM and per iteration: take the largest G that still
            // gives every CTA >= 2 rows and at least one pixel per thread
            int best = G;
            for (int G2 = G + 1; G2 <= SMALL_MAX_CTAS; ++G2) {
                const int R2 = (int)((H + G2 - 1) / G2);
                if (R2 < 2 || (int64_t)(G2 - 1) * R2 >= H) break;
                best = G2;
            }
            *G_out = best;
            *R_out = (int)((H + best - 1) / best);
            return (int64_t)(best - 1) * (*R_out) < H;
        }
    }
    return false;
}

cudaError_t launch_small(const SmallArgs &a, cudaStream_t s) {
    const size_t smem = small_smem_bytes(a.R, a.W);
    cudaError_t e = cudaFuncSetAttribute((const void *)k_small,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (a.G > 8) {
        e = cudaFuncSetAttribute((const void *)k_small,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.G);
    cfg.blockDim = dim3(SMALL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void *args[] = {const_cast<SmallArgs *>(&a)};
    return cudaLaunchKernelExC(&cfg, (const void *)k_small, args);
}

// Can one cluster of G CTAs with this shared memory be scheduled here?
bool small_cluster_fits(const SmallArgs &a) {
    const size_t smem = small_smem_bytes(a.R, a.W);
    if (cudaFuncSetAttribute((const void *)k_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess ||
        (a.G > 8 && cudaFuncSetAttribute((const void *)k_small,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed,
                                         1) != cudaSuccess)) {
        (void)cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.G);
    cfg.blockDim = dim3(SMALL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&n, (const void *)k_small, &cfg) ==
                        cudaSuccess &&
                    n >= 1;
    (void)cudaGetLastError();
    return ok;
}

}  // namespace rds
