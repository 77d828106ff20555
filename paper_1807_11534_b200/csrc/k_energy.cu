// k_energy.cu -- K5: energies and primal-dual gap of the current state (sm_100a).
//
//   TV(w)  = sum |grad w| (forward differences, zero on row H-1 / column W-1)
//   fit(w) = sum f w
//   D(rho) = sum min(0, lambda f + div rho)   (Lagrangian dual of Eq. 4 over u in [0,1])
// for w = v and w = clamp(u, 0, 1).  Per-pixel terms in float32, per-thread/warp/block sums
// in float64; the grid has a fixed size and a fixed pixel -> thread assignment (rows to CTAs,
// columns to threads) and the two passes combine partials in a fixed order, so the result is
// bit-reproducible.
#include "internal.h"

namespace rds {

// |grad| in the energies: MUFU.SQRT (sqrt.approx, relative error < 2^-23, measured:
// profiles/micro_mufu_err.txt); the IEEE sqrtf's slow-path branch made K5 issue-bound.  The
// energies are sums of 10^7 terms compared at 1e-5 relative, far above that error.
__device__ __forceinline__ float esqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int NE = 7;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ float clamp01(float x) { return fminf(fmaxf(x, 0.0f), 1.0f); }

// u' = v_prev - theta div rho (reading R-C12) at pixel (i, j): the last u on RD (the kernel
// wrote exactly that), u0 - theta div rho on pinned pixels (v_prev = u0 there)
__device__ __forceinline__ float u_prime(const EnergyArgs &a, int64_t row, int j) {
    const int64_t o = row + j, os = row + swz(j);
    const uint8_t l = a.lab[o];
    const float dv = a.p1[os] - a.p1[os - a.pitch] + a.p2[os] - a.p2[row + swz(j - 1)];
    return l == 2 ? a.u[o] : (l == 1 ? 1.0f : 0.0f) - a.theta * dv;
}

__global__ void __launch_bounds__(256) k_energy_partial(const EnergyArgs a) {
    const int64_t pitch = a.pitch;
    double acc[NE] = {0, 0, 0, 0, 0, 0, 0};
    // fixed pixel -> thread map: CTA b takes rows row0 + b, row0 + b + G, ...; thread t columns t, t + 256, ...
    for (int i = a.row0 + blockIdx.x; i < a.row1; i += gridDim.x) {
        const int64_t row = (int64_t)i * pitch;
        const bool down = i < a.H - 1;
        int jm = threadIdx.x % a.img_w;  // column within its image (batches)
        for (int j = threadIdx.x; j < a.W; j += 256) {
            const int64_t o = row + j;
            const int64_t os = row + swz(j);  // v, rho are quad-swizzled
            const bool right = jm != a.img_w - 1;
            const float v = a.v[os];
            const float gv1 = down ? a.v[os + pitch] - v : 0.0f;
            const float gv2 = right ? a.v[row + swz(j + 1)] - v : 0.0f;
            const float cu = clamp01(a.u[o]);
            const float gu1 = down ? clamp01(a.u[o + pitch]) - cu : 0.0f;
            const float gu2 = right ? clamp01(a.u[o + 1]) - cu : 0.0f;
            const float f = a.f[o];
            // rho1 on row H-1 and rho2 on an image's last column are identically 0; the frame
            // holds 0
            const float dv = a.p1[os] - a.p1[os - pitch] + a.p2[os] - a.p2[row + swz(j - 1)];
            const float t = a.lambda * f + dv;
            acc[0] += (double)esqrt(gv1 * gv1 + gv2 * gv2);
            acc[1] += (double)f * (double)v;
            acc[2] += (double)esqrt(gu1 * gu1 + gu2 * gu2);
            acc[3] += (double)f * (double)cu;
            acc[4] += (double)fminf(t, 0.0f);
            // F^RD(u', v) = sum_RD |grad u'| + |u' - v|^2 / (2 theta) + lambda <f, v>
            // (branch-free: the band is scattered noise at small delta, so a branch on the
            // label diverges in nearly every warp)
            const uint8_t lx = a.lab[o];  // u' here reuses the div rho of the D term
            const float up = lx == 2 ? a.u[o] : (lx == 1 ? 1.0f : 0.0f) - a.theta * dv;
            const float ud = down ? u_prime(a, row + pitch, j) : up;
            const float ur = right ? u_prime(a, row, j + 1) : up;
            const float g1 = ud - up, g2 = ur - up;
            const float tvp = esqrt(g1 * g1 + g2 * g2);
            acc[5] += (double)(lx == 2 ? tvp : 0.0f);
            acc[6] += (double)((up - v) * (up - v));
            jm += 256;
            while (jm >= a.img_w) jm -= a.img_w;
        }
    }
    __shared__ double sh[8][NE];
#pragma unroll
    for (int q = 0; q < NE; ++q) {
        const double s = warp_sum(acc[q]);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][q] = s;
    }
    __syncthreads();
    if (threadIdx.x < NE) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sh[w][threadIdx.x];
        a.partials[blockIdx.x * NE + threadIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------------------
// Streaming form (round 2): one warp per 120-column strip x row chunk marches down its rows,
// each lane holding a quad of columns (float4 / uchar4 loads: 21 bytes per pixel, every row
// read once; the quad-swizzled v, rho undone in registers).  Lane 0 and lane 31 only supply
// the left / right neighbour quads (the strips overlap by one quad on each side); rows i-1 ..
// i+1 of what the terms need are carried from row to row.  Same per-pixel float terms as
// k_energy_partial; per-warp fp64 sums in a fixed lane order, warps combined in a fixed order
// by k_energy_final, so the result is bit-reproducible.
// ---------------------------------------------------------------------------------------
constexpr int ESTRIP = 120;  // output columns per warp (30 lanes x 4)

struct Q4 {
    float x[4];
};
__device__ __forceinline__ Q4 ld_nat(const float *p) {  // natural-order quad
    const float4 q = *reinterpret_cast<const float4 *>(p);
    return Q4{{q.x, q.y, q.z, q.w}};
}
__device__ __forceinline__ Q4 ld_swz(const float *p) {  // quad-swizzled: x0 x2 x1 x3 in memory
    const float4 q = *reinterpret_cast<const float4 *>(p);
    return Q4{{q.x, q.z, q.y, q.w}};
}

#ifndef RDS_ENERGY_MINB
#define RDS_ENERGY_MINB 1
#endif
__global__ void __launch_bounds__(256, RDS_ENERGY_MINB) k_energy_strip(const EnergyArgs a, int n_strips,
                                                      int chunk, int n_items) {
    const int lane = threadIdx.x & 31;
    const int item = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (item >= n_items) return;  // warp-uniform
    const int s = item % n_strips, c = item / n_strips;
    const int r0 = a.row0 + c * chunk, r1 = min(a.row1, r0 + chunk);
    const int j0 = s * ESTRIP - 4 + 4 * lane;  // this lane's first column
    const bool out_lane = lane >= 1 && lane <= 30;
    const int64_t pitch = a.pitch;
    const float lambda = a.lambda, theta = a.theta;
    // per column: in the image and not an image's last column (grad_2 exists)
    bool inc[4], right[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int j = j0 + e;
        inc[e] = out_lane && j >= 0 && j < a.W;
        right[e] = j >= 0 && j < a.W && (j % a.img_w) != a.img_w - 1;
    }
    auto div_row = [&](const Q4 &p1, const Q4 &p1up, const Q4 &p2, Q4 &d) {
        // div rho = rho1 - rho1(i-1) + rho2 - rho2(j-1); the left neighbour of x0 is the
        // previous lane's x3 (lane 0: its own left quad's value is never used)
        const float l2 = __shfl_up_sync(0xffffffffu, p2.x[3], 1);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            d.x[e] = p1.x[e] - p1up.x[e] + p2.x[e] - (e == 0 ? l2 : p2.x[e - 1]);
    };
    auto uprime = [&](const uchar4 &lb, const Q4 &u, const Q4 &d, Q4 &up) {
        const uint8_t l[4] = {lb.x, lb.y, lb.z, lb.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            up.x[e] = l[e] == 2 ? u.x[e] : (l[e] == 1 ? 1.0f : 0.0f) - theta * d.x[e];
    };
    // row r0 - 1 (rho1 only) and row r0; rows are software-pipelined one ahead: the loads
    // of row i + 2 are in flight while row i's terms are formed (row i + 1's are carried)
    int64_t row = (int64_t)r0 * pitch + j0;
    Q4 p1m = ld_swz(a.p1 + row - pitch);
    Q4 v = ld_swz(a.v + row), p1 = ld_swz(a.p1 + row), p2 = ld_swz(a.p2 + row);
    Q4 u = ld_nat(a.u + row);
    uchar4 lab = *reinterpret_cast<const uchar4 *>(a.lab + row);
    Q4 f = ld_nat(a.f + row);
    // row r0 + 1 (a frame row past H - 1 holds pinned zeros; the chunk's rows are < H)
    Q4 vd = ld_swz(a.v + row + pitch), p1d = ld_swz(a.p1 + row + pitch),
       p2d = ld_swz(a.p2 + row + pitch), ud = ld_nat(a.u + row + pitch);
    uchar4 labd = *reinterpret_cast<const uchar4 *>(a.lab + row + pitch);
    Q4 d, up;
    div_row(p1, p1m, p2, d);
    uprime(lab, u, d, up);
    double acc[NE] = {0, 0, 0, 0, 0, 0, 0};
    for (int i = r0; i < r1; ++i) {
        const bool down = i < a.H - 1;
        const int64_t rn = row + pitch, rnn = rn + pitch;
        // prefetch row i + 2 (and f of row i + 1); rows past the frame are not read
        const bool pre = i + 2 <= a.H && i + 1 < r1;
        Q4 vn, p1n, p2n, un, fn;
        uchar4 labn = make_uchar4(0, 0, 0, 0);
        if (pre) {
            vn = ld_swz(a.v + rnn);
            p1n = ld_swz(a.p1 + rnn);
            p2n = ld_swz(a.p2 + rnn);
            un = ld_nat(a.u + rnn);
            labn = *reinterpret_cast<const uchar4 *>(a.lab + rnn);
        }
        if (i + 1 < r1) fn = ld_nat(a.f + rn);
        Q4 dd, upd;
        div_row(p1d, p1, p2d, dd);
        uprime(labd, ud, dd, upd);
        // right neighbours of x3: the next lane's x0
        const float vr = __shfl_down_sync(0xffffffffu, v.x[0], 1);
        const float ur = __shfl_down_sync(0xffffffffu, u.x[0], 1);
        const float upr = __shfl_down_sync(0xffffffffu, up.x[0], 1);
        const uint8_t l[4] = {lab.x, lab.y, lab.z, lab.w};
        // the row's four columns are summed in fp32 (selects, no branches), then once in fp64
        float r[NE] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float vx = v.x[e], ux = u.x[e], fx = f.x[e];
            const float vnext = e < 3 ? v.x[e + 1] : vr;
            const float unext = e < 3 ? u.x[e + 1] : ur;
            const float upnext = e < 3 ? up.x[e + 1] : upr;
            const float gv1 = down ? vd.x[e] - vx : 0.0f;
            const float gv2 = right[e] ? vnext - vx : 0.0f;
            const float cu = clamp01(ux);
            const float gu1 = down ? clamp01(ud.x[e]) - cu : 0.0f;
            const float gu2 = right[e] ? clamp01(unext) - cu : 0.0f;
            const float t = lambda * fx + d.x[e];
            const float upx = up.x[e];
            const float g1 = (down ? upd.x[e] : upx) - upx;
            const float g2 = (right[e] ? upnext : upx) - upx;
            const float tvp = esqrt(g1 * g1 + g2 * g2);
            const bool in = inc[e];
            r[0] += in ? esqrt(gv1 * gv1 + gv2 * gv2) : 0.0f;
            r[1] += in ? fx * vx : 0.0f;
            r[2] += in ? esqrt(gu1 * gu1 + gu2 * gu2) : 0.0f;
            r[3] += in ? fx * cu : 0.0f;
            r[4] += in ? fminf(t, 0.0f) : 0.0f;
            r[5] += in && l[e] == 2 ? tvp : 0.0f;
            r[6] += in ? (upx - vx) * (upx - vx) : 0.0f;
        }
#pragma unroll
        for (int q = 0; q < NE; ++q) acc[q] += (double)r[q];
        // carry rows i + 1 and i + 2
        p1m = p1;
        v = vd;
        p1 = p1d;
        p2 = p2d;
        u = ud;
        lab = labd;
        d = dd;
        up = upd;
        f = fn;
        vd = vn;
        p1d = p1n;
        p2d = p2n;
        ud = un;
        labd = labn;
        row = rn;
    }
#pragma unroll
    for (int q = 0; q < NE; ++q) {
        const double sum = warp_sum(acc[q]);
        if (lane == 0) a.partials[(int64_t)item * NE + q] = sum;
    }
}

__global__ void __launch_bounds__(256) k_energy_final(const double *partials, int nb,
                                                      double *out) {
    __shared__ double sh[8][NE];
    double acc[NE] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nb; b += 256)
#pragma unroll
        for (int q = 0; q < NE; ++q) acc[q] += partials[b * NE + q];
#pragma unroll
    for (int q = 0; q < NE; ++q) {
        const double s = warp_sum(acc[q]);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5][q] = s;
    }
    __syncthreads();
    if (threadIdx.x < NE) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sh[w][threadIdx.x];
        out[threadIdx.x] = s;
    }
}

__global__ void k_unswizzle(const float *plane, int64_t pitch, int H, int W, float *out,
                            int64_t out_pitch) {
    const int64_t n = (int64_t)H * W;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(k / W), j = (int)(k - (int64_t)i * W);
        out[(int64_t)i * out_pitch + j] = plane[(int64_t)i * pitch + swz(j)];
    }
}

template <typename T>
__global__ void k_batch_copy(T *dense, T *plane, int64_t pitch, int H, int iw, int B,
                             int to_plane, int swizzled) {
    const int64_t n = (int64_t)B * H * iw;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bh = k / iw;
        const int j = (int)(k - bh * iw);
        const int b = (int)(bh / H), i = (int)(bh - (int64_t)b * H);
        const int col = b * iw + j;
        const int64_t o = (int64_t)i * pitch + (swizzled ? swz(col) : col);
        if (to_plane)
            plane[o] = dense[k];
        else
            dense[k] = plane[o];
    }
}

cudaError_t launch_batch_copy(void *dense, void *plane, int elt, int64_t pitch, int H,
                              int img_w, int B, int to_plane, int swizzled, cudaStream_t s) {
    if (elt == 8)
        k_batch_copy<double><<<148 * 8, 256, 0, s>>>((double *)dense, (double *)plane, pitch, H,
                                                      img_w, B, to_plane, swizzled);
    else if (elt == 4)
        k_batch_copy<float><<<148 * 8, 256, 0, s>>>((float *)dense, (float *)plane, pitch, H,
                                                     img_w, B, to_plane, swizzled);
    else
        k_batch_copy<uint8_t><<<148 * 8, 256, 0, s>>>((uint8_t *)dense, (uint8_t *)plane, pitch,
                                                       H, img_w, B, to_plane, swizzled);
    return cudaGetLastError();
}

// Frame integrity (a memory-safety check that needs no sanitizer): every element of a padded
// plane outside the H x W image must still hold the pinned frame value it was allocated with.
// Counts the elements that differ (natural-order column index mapped through the swizzle for
// swizzled planes).
template <typename T>
__global__ void k_frame_check(const T *base, int64_t pitch, int64_t rows, int64_t origin_row,
                              int64_t origin_col, int H, int W, int swizzled, T expect,
                              unsigned long long *bad) {
    const int64_t n = rows * pitch;
    unsigned long long cnt = 0;
    // k enumerates LOGICAL positions (row r, column c of the padded plane); a frame position
    // (outside the image) is looked up where it is stored: column c itself, or its swizzled
    // column for quad-swizzled planes (the swizzle stays inside an aligned quad)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = k / pitch, c = k - r * pitch;
        const int64_t i = r - origin_row, j = c - origin_col;
        if (i >= 0 && i < H && j >= 0 && j < W) continue;  // image element
        const int64_t cc = (swizzled ? (int64_t)swz((int)j) : j) + origin_col;
        if (!(base[r * pitch + cc] == expect)) ++cnt;
    }
    if (cnt) atomicAdd(bad, cnt);
}

cudaError_t launch_frame_check(const void *base, int elt, int64_t pitch, int64_t rows,
                               int64_t origin_row, int64_t origin_col, int H, int W,
                               int swizzled, double expect, unsigned long long *bad,
                               cudaStream_t s) {
    if (elt == 4)
        k_frame_check<float><<<148 * 4, 256, 0, s>>>((const float *)base, pitch, rows,
                                                      origin_row, origin_col, H, W, swizzled,
                                                      (float)expect, bad);
    else
        k_frame_check<uint8_t><<<148 * 4, 256, 0, s>>>((const uint8_t *)base, pitch, rows,
                                                        origin_row, origin_col, H, W, swizzled,
                                                        (uint8_t)expect, bad);
    return cudaGetLastError();
}

cudaError_t launch_unswizzle(const float *plane, int64_t pitch, int H, int W, float *out,
                             int64_t out_pitch, cudaStream_t s) {
    k_unswizzle<<<148 * 8, 256, 0, s>>>(plane, pitch, H, W, out, out_pitch);
    return cudaGetLastError();
}

cudaError_t launch_energy(const EnergyArgs &a, cudaStream_t s) {
    // strips of ESTRIP columns x row chunks, at most ENERGY_WARPS warps (the partials buffer)
    const int n_strips = (a.W + ESTRIP - 1) / ESTRIP;
    const int rows = a.row1 - a.row0;
    if (rows <= 0 || n_strips <= 0) {
        k_energy_final<<<1, 256, 0, s>>>(a.partials, 0, a.out);
        return cudaGetLastError();
    }
    int chunks = ENERGY_WARPS / n_strips;
    if (chunks < 1) chunks = 1;
    int chunk = (rows + chunks - 1) / chunks;
    if (chunk < 16) chunk = 16;  // short chunks: the first-row loads would dominate
    chunks = (rows + chunk - 1) / chunk;
    if ((int64_t)chunks * n_strips > ENERGY_WARPS) {  // very wide images: the old kernel
        k_energy_partial<<<ENERGY_BLOCKS, 256, 0, s>>>(a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        k_energy_final<<<1, 256, 0, s>>>(a.partials, ENERGY_BLOCKS, a.out);
        return cudaGetLastError();
    }
    const int n_items = chunks * n_strips;
    k_energy_strip<<<(n_items + 7) / 8, 256, 0, s>>>(a, n_strips, chunk, n_items);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_energy_final<<<1, 256, 0, s>>>(a.partials, n_items, a.out);
    return cudaGetLastError();
}

}  // namespace rds

namespace rds {

// Stopping rule of PAPER.md:234-238, max{||u^l - u^(l-1)||, ||v^l - v^(l-1)||} <= tol
// (reading R-F2: Euclidean norm over pixels of unit area, or RMS): one CTA sums the block's
// per-item (or per-CTA) partials in a fixed order (thread-strided sums, then a fixed tree),
// so the decision is deterministic.  Pinned pixels contribute 0.  Every check advances the
// record's iteration / launch counters; inside a CUDA-graph while loop the body's last check
// also sets the loop condition.
__global__ void __launch_bounds__(256) k_stop_check(const StopCheck c) {
    StopRecord *rec = c.rec;
    if (*(volatile const int32_t *)&rec->flag != 0) {  // uniform across the CTA
        if (c.set_cond && threadIdx.x == 0) cudaGraphSetConditional(c.cond, 0);
        return;
    }
    const int n = *c.n_part;
    double su = 0.0, sv = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) {
        su += c.part[2 * i];
        sv += c.part[2 * i + 1];
    }
    __shared__ double sh[2][8];
    su = warp_sum(su);
    sv = warp_sum(sv);
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = su;
        sh[1][threadIdx.x >> 5] = sv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tu = 0.0, tv = 0.0;
        for (int w = 0; w < 8; ++w) {
            tu += sh[0][w];
            tv += sh[1][w];
        }
        const double r = fmax(sqrt(tu / c.norm_div), sqrt(tv / c.norm_div));
        rec->su = tu;
        rec->sv = tv;
        const int it = rec->it + c.block_iters;
        rec->it = it;
        rec->launches += c.block_launches;
        rec->residual = r;
        rec->checks += 1;
        const bool conv = r <= c.tol;
        const bool fire = conv || it >= c.max_iters;
        if (fire) {
            rec->iters = it;
            rec->converged = conv ? 1 : 0;
            rec->flag = 1;
        }
        if (c.set_cond)
            cudaGraphSetConditional(c.cond, (!fire && it + c.body_iters <= c.loop_end) ? 1 : 0);
    }
}

cudaError_t launch_stop_check(const StopCheck &c, cudaStream_t s) {
    k_stop_check<<<1, 256, 0, s>>>(c);
    return cudaGetLastError();
}

}  // namespace rds
