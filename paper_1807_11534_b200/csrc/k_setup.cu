// k_setup.cu -- per-solve setup kernels of librds (sm_100a):
//   K1 k_setup      fused fitting term + band test + initialisation + per-tile RD counts
//   K2 k_compact    warp-ballot / prefix-sum compaction of the active-tile list
//      k_band_flags / k_build_items: stencil work items = runs of active 32-row bands per
//                   column strip, split into near-equal pieces
//   plus the absmax reduction (delta = delta_rel * max|f|) and the finiteness check.
//
// PAPER.md references: fitting term Eq. 2-3; partition;
// initialisation u0 = H(-f), rho0 = 0; v0 = u0 (reading R-C9).
#include <math.h>

#include "internal.h"

namespace rds {

// f = (z - c1)^2 - (z - c2)^2 (+ gamma P): float32 with a fixed operation order and no
// contraction (explicit _rn intrinsics), so labels are bit-identical to the oracle's
// (reading R-A1).
__device__ __forceinline__ float fitting_term(float z, float P, float c1, float c2,
                                              float gamma, bool use_p) {
    float a = __fsub_rn(z, c1);
    float b = __fsub_rn(z, c2);
    float f = __fsub_rn(__fmul_rn(a, a), __fmul_rn(b, b));
    if (use_p) f = __fadd_rn(f, __fmul_rn(gamma, P));
    return f;
}

__global__ void k_fill(float *p, int64_t n, float value) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        p[k] = value;
}

cudaError_t launch_fill_frame(float *plane, int64_t n, float value, cudaStream_t s) {
    int grid = (int)((n + 255) / 256);
    if (grid > 148 * 32) grid = 148 * 32;
    k_fill<<<grid, 256, 0, s>>>(plane, n, value);
    return cudaGetLastError();
}

__global__ void k_check_finite(const float *a, int64_t pitch, int H, int W, int *flag) {
    int64_t n = (int64_t)H * W;
    int bad = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = k / W, j = k - i * W;
        if (!isfinite(a[i * pitch + j])) bad = 1;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t launch_check_finite(const float *a, int64_t pitch, int H, int W, int *flag,
                                cudaStream_t s) {
    k_check_finite<<<148 * 4, 256, 0, s>>>(a, pitch, H, W, flag);
    return cudaGetLastError();
}

// max |f| as the bit pattern of a non-negative float (uint order == float order), so the
// atomic max is order-independent and the result deterministic.
__global__ void k_absmax(const float *z, const float *P, int64_t pitch, int H, int W,
                         float c1, float c2, float gamma, unsigned *out_bits) {
    int64_t n = (int64_t)H * W;
    bool use_p = gamma != 0.0f;
    float m = 0.0f;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = k / W, j = k - i * W;
        int64_t o = i * pitch + j;
        float f = fitting_term(z[o], use_p ? P[o] : 0.0f, c1, c2, gamma, use_p);
        m = fmaxf(m, fabsf(f));
    }
    for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(m));
}

cudaError_t launch_absmax(const float *z, const float *P, int64_t pitch, int H, int W,
                          float c1, float c2, float gamma, unsigned *out_bits,
                          cudaStream_t s) {
    k_absmax<<<148 * 4, 256, 0, s>>>(z, P, pitch, H, W, c1, c2, gamma, out_bits);
    return cudaGetLastError();
}

// Radix-select pass for the q -> q^ search: histogram of byte `shift` of the
// bit pattern of |f| over the pixels whose higher bytes equal `prefix` (under `mask`).
// Non-negative floats order like their bit patterns, so 4 passes find the k-th smallest |f|
// exactly; integer counts make the result independent of the atomic order.
__global__ void k_abs_hist(const float *z, const float *P, int64_t pitch, int H, int W,
                           float c1, float c2, float gamma, unsigned prefix, unsigned mask,
                           int shift, unsigned *hist) {
    __shared__ unsigned sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t n = (int64_t)H * W;
    const bool use_p = gamma != 0.0f;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k / W, j = k - i * W, o = i * pitch + j;
        const float f = fitting_term(z[o], use_p ? P[o] : 0.0f, c1, c2, gamma, use_p);
        const unsigned b = __float_as_uint(fabsf(f));
        if ((b & mask) == prefix) atomicAdd(&sh[(b >> shift) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

cudaError_t launch_abs_hist(const float *z, const float *P, int64_t pitch, int H, int W,
                            float c1, float c2, float gamma, unsigned prefix, unsigned mask,
                            int shift, unsigned *hist, cudaStream_t s) {
    k_abs_hist<<<148 * 4, 256, 0, s>>>(z, P, pitch, H, W, c1, c2, gamma, prefix, mask, shift,
                                        hist);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// K1: one CTA per 32x32 tile, 256 threads, 4 consecutive pixels (one float4) per thread.
// Writes f, the label byte, c' (2^-100 theta*lambda*f on RD, -inf on Fg, +inf on Bg), u = mask = u0,
// and the initial state into BOTH ping-pong buffers (c', rho and v quad-swizzled, internal.h;
// pinned pixels never change, and a
// skipped work item must read as its initial value from either buffer).  Out-of-image
// columns of the tile are written with the frame's pinned values (rho = 0, v = 0, c = +inf).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_setup(SetupArgs a) {
    const int r = threadIdx.x >> 3;           // row in tile
    const int q = threadIdx.x & 7;            // float4 column group in tile
    const int i = blockIdx.y * TILE_H + r;
    const int j = blockIdx.x * TILE_W + 4 * q;
    const bool use_p = a.gamma != 0.0f;
    int rd_count = 0;
    if (i < a.H) {
        const int64_t o = (int64_t)i * a.pitch + j;
        const float4 z4 = *reinterpret_cast<const float4 *>(a.z + o);
        float4 P4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (use_p) P4 = *reinterpret_cast<const float4 *>(a.P + o);
        float4 wv4 = P4, wp14 = P4, wp24 = P4;
        if (a.wv) {
            wv4 = *reinterpret_cast<const float4 *>(a.wv + o);
            wp14 = *reinterpret_cast<const float4 *>(a.wp1 + o);
            wp24 = *reinterpret_cast<const float4 *>(a.wp2 + o);
        }
        const float zz[4] = {z4.x, z4.y, z4.z, z4.w};
        const float PP[4] = {P4.x, P4.y, P4.z, P4.w};
        const float WV[4] = {wv4.x, wv4.y, wv4.z, wv4.w};
        const float W1[4] = {wp14.x, wp14.y, wp14.z, wp14.w};
        const float W2[4] = {wp24.x, wp24.y, wp24.z, wp24.w};
        float f[4], c[4], v[4], p1[4], p2[4], u[4];
        uint8_t lab[4], msk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int jj = j + e;
            if (jj < a.W) {
                const float fe = fitting_term(zz[e], PP[e], a.c1, a.c2, a.gamma, use_p);
                const bool rd = fabsf(fe) < a.delta;           // RD <=> |f| < delta
                const bool fg = fe <= 0.0f;                    // H(-f), H(0) = 1
                const float u0 = fg ? 1.0f : 0.0f;
                f[e] = fe;
                lab[e] = rd ? 2 : (fg ? 1 : 0);
                // RD: theta*lambda*f clamped to +-2^20 (the v-step saturates far earlier:
                // |u| <= max|v| + 4 theta) and stored as c' = c * 2^-100, so |c'| <= 2^-80
                // is negligible under the stencil's square root (k_stencil_impl.cuh, stage()).
                c[e] = rd ? __fmul_rn(fminf(fmaxf(__fmul_rn(a.theta_lambda, fe), -0x1p20f),
                                            0x1p20f),
                                      0x1p-100f)
                          : (fg ? -INFINITY : INFINITY);
                u[e] = u0;
                msk[e] = fg ? 1 : 0;
                const bool warm = rd && a.wv != nullptr;
                v[e] = warm ? WV[e] : u0;
                p1[e] = (warm && i < a.H - 1) ? W1[e] : 0.0f;
                p2[e] = (warm && jj % a.img_w != a.img_w - 1) ? W2[e] : 0.0f;
                rd_count += rd;
            } else {
                f[e] = 0.0f;
                lab[e] = 0;
                c[e] = INFINITY;
                u[e] = 0.0f;
                msk[e] = 0;
                v[e] = 0.0f;
                p1[e] = 0.0f;
                p2[e] = 0.0f;
            }
        }
        *reinterpret_cast<float4 *>(a.f + o) = make_float4(f[0], f[1], f[2], f[3]);
        *reinterpret_cast<float4 *>(a.u + o) = make_float4(u[0], u[1], u[2], u[3]);
        // the stencil's state planes are quad-swizzled (internal.h): memory x0 x2 x1 x3
        *reinterpret_cast<float4 *>(a.c + o) = make_float4(c[0], c[2], c[1], c[3]);
        const float4 v4 = make_float4(v[0], v[2], v[1], v[3]);
        const float4 p14 = make_float4(p1[0], p1[2], p1[1], p1[3]);
        const float4 p24 = make_float4(p2[0], p2[2], p2[1], p2[3]);
        *reinterpret_cast<float4 *>(a.v0 + o) = v4;
        *reinterpret_cast<float4 *>(a.v1 + o) = v4;
        *reinterpret_cast<float4 *>(a.p10 + o) = p14;
        *reinterpret_cast<float4 *>(a.p11 + o) = p14;
        *reinterpret_cast<float4 *>(a.p20 + o) = p24;
        *reinterpret_cast<float4 *>(a.p21 + o) = p24;
        *reinterpret_cast<uchar4 *>(a.lab + o) = make_uchar4(lab[0], lab[1], lab[2], lab[3]);
        *reinterpret_cast<uchar4 *>(a.mask + o) = make_uchar4(msk[0], msk[1], msk[2], msk[3]);
    }
    // per-tile RD count (deterministic integer sum)
    __shared__ int warp_sum[8];
    int s = __reduce_add_sync(0xffffffffu, rd_count);
    if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        const int tile = blockIdx.y * gridDim.x + blockIdx.x;
        int t = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += warp_sum[w];
        a.tile_rd[tile] = t;
        // warp w holds rows 4w..4w+3, so the 8-row sub-tile k is warps 2k, 2k+1
#pragma unroll
        for (int k = 0; k < SUBTILES; ++k) a.sub_rd[tile * SUBTILES + k] = warp_sum[2 * k] + warp_sum[2 * k + 1];
    }
}

cudaError_t launch_setup(const SetupArgs &a, cudaStream_t s) {
    dim3 grid((a.W + TILE_W - 1) / TILE_W, (a.H + TILE_H - 1) / TILE_H);
    k_setup<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// K2: single-CTA compaction.  Each round covers 1024 flags: __ballot_sync + __popc give the
// rank inside the warp, a shuffle scan over the 32 warp totals gives the warp offsets, so
// the output list is in ascending index order and identical on every run (no atomics).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_compact(const int32_t *flags, int n, int32_t *list,
                                                  int32_t *count, long long *sum_out) {
    __shared__ int warp_off[32];
    __shared__ int round_total;
    __shared__ long long warp_sum[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int base = 0;
    long long mysum = 0;
    for (int start = 0; start < n; start += 1024) {
        const int i = start + tid;
        const int val = (i < n) ? flags[i] : 0;
        mysum += val;
        const bool on = val != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        const int rank = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) warp_off[wid] = __popc(bal);
        __syncthreads();
        if (wid == 0) {
            const int t = warp_off[lane];
            int incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            warp_off[lane] = incl - t;
            if (lane == 31) round_total = incl;
        }
        __syncthreads();
        if (on) list[base + warp_off[wid] + rank] = i;
        base += round_total;
        __syncthreads();
    }
    if (tid == 0) *count = base;
    if (sum_out) {
        for (int o = 16; o; o >>= 1) mysum += __shfl_xor_sync(0xffffffffu, mysum, o);
        if (lane == 0) warp_sum[wid] = mysum;
        __syncthreads();
        if (tid == 0) {
            long long t = 0;
            for (int w = 0; w < 32; ++w) t += warp_sum[w];
            *sum_out = t;
        }
    }
}

cudaError_t launch_compact(const int32_t *flags, int n, int32_t *list, int32_t *count,
                           long long *sum_out, cudaStream_t s) {
    k_compact<<<1, 1024, 0, s>>>(flags, n, list, count, sum_out);
    return cudaGetLastError();
}

// A strip's band b (BAND_H = 8 rows) is active iff one of the 32-column x 8-row sub-tiles
// its output columns overlap in that band holds an RD pixel.  Processing a pinned pixel
// reproduces its value exactly, so any superset of the needed work gives the same result;
// skip = 0 marks every band active.
__global__ void k_band_flags(const int32_t *sub_rd, int H, int W, int wv, int n_strips,
                             int skip, uint32_t *band_bits) {
    const int n_bands = (H + BAND_H - 1) / BAND_H, nbw = (n_bands + 31) / 32;
    const int it = blockIdx.x * blockDim.x + threadIdx.x;  // s * nbw * 32 + b: a warp = one word
    if (it >= n_strips * nbw * 32) return;                  // whole warps only (see launch)
    const int s = it / (nbw * 32), b = it - s * nbw * 32;
    int on = 0;
    if (b < n_bands) {
        if (!skip) {
            on = 1;
        } else {
            const int ntj = (W + TILE_W - 1) / TILE_W;
            const int ti = b / SUBTILES, k = b - ti * SUBTILES;
            const int j0 = s * wv, j1 = min(W, (s + 1) * wv) - 1;
            for (int tj = j0 / TILE_W; tj <= j1 / TILE_W; ++tj)
                on |= sub_rd[(ti * ntj + tj) * SUBTILES + k] != 0;
        }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 31) == 0) band_bits[it >> 5] = word;
}

cudaError_t launch_band_flags(const int32_t *sub_rd, int H, int W, int wv, int n_strips,
                              int skip, uint32_t *band_bits, cudaStream_t s) {
    const int nbw = ((H + BAND_H - 1) / BAND_H + 31) / 32;
    const int n = n_strips * nbw * 32;  // a multiple of 32: every warp is complete
    k_band_flags<<<(n + 255) / 256, 256, 0, s>>>(sub_rd, H, W, wv, n_strips, skip, band_bits);
    return cudaGetLastError();
}

// Item rows are cut at multiples of ITEM_Q rows (finer than a 32-row band), so a sparse
// active set, or a dense one that would overflow the resident warps by a few items, can be
// spread over every warp.  Candidate item heights (rows) for the makespan model:

__constant__ int kChunkRows[] = {8, 16, 24, 32, 40, 48, 64, 80, 96, 128, 160, 192, 256, 384, 512};
constexpr int N_CHUNK = 15;

// Runs of active bands in strip s (rows clipped to H), split into ceil(rows / chunk) pieces of
// near-equal height at ITEM_Q-row boundaries; out == nullptr only counts.
__device__ int strip_items(const uint32_t *bits, int nbw, int H, int chunk, int s, Item *out) {
    int n = 0, pos = 0, b, e;
    while (next_run(bits, nbw, &pos, &b, &e)) {
        const int r0 = b * BAND_H, r1 = min(e * BAND_H, H);
        const int q = (r1 - r0 + ITEM_Q - 1) / ITEM_Q;            // ITEM_Q-row slices
        const int pieces = (r1 - r0 + chunk - 1) / chunk;
        for (int k = 0; k < pieces; ++k) {
            if (out) {
                const int p0 = r0 + ITEM_Q * (int)((int64_t)k * q / pieces);
                const int p1 = min(r1, r0 + ITEM_Q * (int)((int64_t)(k + 1) * q / pieces));
                out[n] = Item{s, p0, p1, 0};
            }
            ++n;
        }
    }
    return n;
}

// Single CTA.  (1) For every candidate height c, the exact item count sum over runs of
// ceil(rows / c); the makespan model picks the c minimising
//     (waves - 1) * (hbar + w) + (c + w),   waves = ceil(items / resident warps),
// hbar = active rows / items (the mean item height, below c when runs are short), w = the
// pipeline warm-up rows: whole rounds of items (one extra item on a full wave doubles the
// launch), the last round set by the tallest item; ties go to the taller item.
// (2) Per-strip item counts -> block exclusive scan -> items written in strip-major,
// ascending-row order (deterministic, no atomics).
__global__ void __launch_bounds__(1024) k_build_items(const uint32_t *band_bits, int n_strips,
                                                      int n_bands, int H, int slots,
                                                      int fixed_chunk, int max_chunk,
                                                      int warmup_rows, Item *items,
                                                      int32_t *counts) {
    __shared__ long long red[N_CHUNK + 2][32];
    __shared__ int off[32];
    __shared__ int chunk_s, base_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    long long cnt_c[N_CHUNK + 2];  // items per candidate, active cells, active rows
#pragma unroll
    for (int k = 0; k <= N_CHUNK + 1; ++k) cnt_c[k] = 0;
    const int nbw = (n_bands + 31) / 32;
    for (int sidx = tid; sidx < n_strips; sidx += 1024) {
        const uint32_t *bits = band_bits + (int64_t)sidx * nbw;
        int pos = 0, b, e;
        while (next_run(bits, nbw, &pos, &b, &e)) {
            const int rows = min(e * BAND_H, H) - b * BAND_H;
#pragma unroll
            for (int k = 0; k < N_CHUNK; ++k) cnt_c[k] += (rows + kChunkRows[k] - 1) / kChunkRows[k];
            cnt_c[N_CHUNK] += e - b;  // active cells
            cnt_c[N_CHUNK + 1] += rows;
        }
    }
#pragma unroll
    for (int k = 0; k <= N_CHUNK + 1; ++k) {
        long long v = cnt_c[k];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[k][wid] = v;
    }
    __syncthreads();
    if (tid == 0) {
        int c = fixed_chunk > 0 ? (fixed_chunk + ITEM_Q - 1) / ITEM_Q * ITEM_Q : 0;
        if (c > max_chunk) c = max_chunk;
        if (c <= 0) {
            const long long sl = slots > 0 ? slots : 1;
            long long rows_all = 0;
            for (int w = 0; w < 32; ++w) rows_all += red[N_CHUNK + 1][w];
            double best = -1.0;
            for (int k = 0; k < N_CHUNK; ++k) {
                if (kChunkRows[k] > max_chunk && k > 0) continue;
                long long items_k = 0;
                for (int w = 0; w < 32; ++w) items_k += red[k][w];
                const long long waves = (items_k + sl - 1) / sl;
                const double hbar = items_k > 0 ? (double)rows_all / (double)items_k : 0.0;
                const double cost = (double)(waves > 1 ? waves - 1 : 0) * (hbar + warmup_rows) +
                                    (double)(kChunkRows[k] + warmup_rows);
                if (best < 0.0 || cost <= best) {
                    best = cost;
                    c = kChunkRows[k];
                }
            }
        }
        chunk_s = c;
        base_s = 0;
    }
    __syncthreads();
    const int chunk = chunk_s;
    for (int s0 = 0; s0 < n_strips; s0 += 1024) {
        const int sidx = s0 + tid;
        const int cnt = sidx < n_strips ? strip_items(band_bits + (int64_t)sidx * nbw, nbw, H,
                                                      chunk, sidx, nullptr)
                                        : 0;
        // block exclusive scan of cnt
        int incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) off[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int t = off[lane];
            int in2 = t;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, in2, o);
                if (lane >= o) in2 += y;
            }
            off[lane] = in2 - t;
        }
        __syncthreads();
        const int start = base_s + off[wid] + incl - cnt;
        if (sidx < n_strips)
            strip_items(band_bits + (int64_t)sidx * nbw, nbw, H, chunk, sidx, items + start);
        __syncthreads();
        if (tid == 1023) base_s = start + cnt;
        __syncthreads();
    }
    if (tid == 0) {
        counts[1] = base_s;
        counts[2] = chunk;
        long long t = 0;
        for (int w = 0; w < 32; ++w) t += red[N_CHUNK][w];
        counts[3] = (int32_t)t;
    }
}

cudaError_t launch_build_items(const uint32_t *band_bits, int n_strips, int n_bands, int H,
                               int slots, int fixed_chunk, int max_chunk, int warmup_rows,
                               Item *items, int32_t *counts, cudaStream_t s) {
    k_build_items<<<1, 1024, 0, s>>>(band_bits, n_strips, n_bands, H, slots, fixed_chunk,
                                     max_chunk, warmup_rows, items, counts);
    return cudaGetLastError();
}

}  // namespace rds
