// k_grid.cu -- mid-size images (up to about 10^6 pixels: C1's 1024 x 1024) resident on the
// whole GPU: the K-loop of a fixed-K solve in ONE cooperative launch, the state in registers
// of G <= #SM co-resident CTAs, the slab halos exchanged every iteration through an L2
// mailbox of {value, tag} words -- no grid barrier, no flag, no fence: each thread polls the
// words of its own columns that its two neighbour slabs publish (DESIGN.md §5 "resident grid").
//
// The image is cut into G horizontal slabs of R rows (R a compile-time 2 .. 8), one CTA each
// (one CTA per SM: 512 threads x <= 128 registers).  A thread owns TWO adjacent columns
// j0 = 2t, j1 = 2t + 1 of its slab and keeps their state in registers: rho1, rho2, v and c'
// for local rows -2 .. R (the halo rows -2, -1 above and R below belong to the neighbour
// slabs).  Iteration k is the one of k_small.cu (Eq. 7-9, the rho fixed
// point of PAPER.md:138-141), phases
//   A  w = div rho - v / theta             rows -1 .. R
//   B  rho' = (rho + tau grad w) rr        rows -1 .. R-1 (in place: rho of a row is dead once
//                                           the w that read it exist)
//   C  u = v - theta div rho', v' = sat(u - c)  rows 0 .. R-1
// each split into the rows that need no halo (done first) and the boundary rows (done after
// the neighbours' rows of iteration k - 1 arrived), then the slab's new rows 0 and R-2, R-1
// are published.  Row -1's rho' is recomputed here bit-identically to the neighbour's.
// The column pair's left neighbour (column 2t - 1) is the previous lane's x1, its right one
// (2t + 2) the next lane's x0 (shuffles); warp-edge columns go through shared memory (four
// CTA barriers per iteration).  Every float operation is the one k_stencil performs, in the
// same order: the result equals the stencil's bit for bit.
//
// Mailbox reuse is safe with two parities: a thread overwrites its words of slot k & 1 at
// iteration k + 2 only after it read its neighbours' words of iteration k + 1, which they
// published after reading slot k & 1 at iteration k (and after the CTA barriers that order
// every read of their iteration k).  Tags grow across launches (tag0, set by the host), so a
// word left by an earlier solve never matches.  All G CTAs must be co-resident (cooperative
// launch; the launcher checks the occupancy); a wait that never ends traps instead of hanging.
#include <cooperative_groups.h>
#include <cstdio>
#include <math.h>

#include "internal.h"

namespace rds {

namespace {

__device__ __forceinline__ float sqrt_gx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_gx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Mailbox entries are {value, tag} pairs in one 8-byte word: an aligned 8-byte access is
// single-copy atomic, so a reader that sees the tag it waits for sees the value with it -- no
// fence, no flag, every thread polls exactly the words it needs (L2, relaxed gpu scope).
__device__ __forceinline__ unsigned long long ll_pack(float x, unsigned tag) {
    return ((unsigned long long)tag << 32) | __float_as_uint(x);
}
__device__ __forceinline__ void ll_st2(unsigned long long *p, float2 x, unsigned tag) {
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(ll_pack(x.x, tag)),
                 "l"(ll_pack(x.y, tag))
                 : "memory");
}
__device__ __forceinline__ void ll_ld2(const unsigned long long *p, unsigned long long &x,
                                       unsigned long long &y) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                 : "=l"(x), "=l"(y)
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ unsigned long long ll_ld1(const unsigned long long *p) {
    unsigned long long x;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ bool ll_ok(unsigned long long x, unsigned tag) {
    return (unsigned)(x >> 32) == tag;
}
__device__ __forceinline__ float ll_val(unsigned long long x) {
    return __uint_as_float((unsigned)x);
}
// wait for two {value, tag} words (a column pair) of the given tag
__device__ __forceinline__ float2 ll_wait2(const unsigned long long *p, unsigned tag) {
    unsigned long long x, y;
    unsigned long long spins = 0;
    for (;;) {
        ll_ld2(p, x, y);
        if (ll_ok(x, tag) && ll_ok(y, tag)) break;
        if (++spins > (1ull << 31)) __trap();  // cannot happen with co-resident CTAs
    }
    return make_float2(ll_val(x), ll_val(y));
}

constexpr unsigned FULL = 0xffffffffu;
constexpr int GRID_THREADS = 512;
#ifndef RDS_GRID_BACKOFF
#define RDS_GRID_BACKOFF (void)0
#endif

}  // namespace

// Mailbox slot of CTA g at parity p: 7 rows of NC = 2 * blockDim {value, tag} words
//   0 rho1(R-2), 1 rho1(R-1), 2 rho1(0), 3 rho2(R-1), 4 rho2(0), 5 v(R-1), 6 v(0)
// (rows 0, 1, 3, 5 are the CTA below's halo rows -2, -1; rows 2, 4, 6 the CTA above's row R),
// published at iteration k with tag tag0 + k.
//
// Each iteration runs the rows that need no halo first (interior: w on rows 1 .. R-1, rho' on
// 1 .. R-2, u / v' on 2 .. R-2), then waits for the neighbours' rows of the previous
// iteration, then the boundary rows (w on -1, 0, R; rho' on -1, 0, R-1; u / v' on 0, 1, R-1)
// and publishes: the exchange latency hides behind the interior work.  In local indices
// r = row + 2 (0 .. NR-1): interior A r = 3 .. R+1, B r = 3 .. R, C r = 4 .. R; boundary
// A r = 1, 2, NR-1, B r = 1, 2, R+1, C r = 2, 3, R+1.
template <int R>
__global__ void __launch_bounds__(GRID_THREADS, 1) k_grid(const GridArgs a) {
    constexpr int NR = R + 3;
    // warp-edge columns: lane 0's w (for the warp to the left), lane 31's rho2 (to the right)
    __shared__ float eW[GRID_THREADS / 32][NR], eP[GRID_THREADS / 32][NR];
    const int NT = blockDim.x, NW = NT >> 5, NC = 2 * NT;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int rank = blockIdx.x, G = a.G;
    const int r0 = rank * R, H = a.H, W = a.W;
    const int j0 = 2 * t, j1 = j0 + 1;
    const bool ok0 = j0 < W, ok1 = j1 < W;
    const bool g2z0 = !ok0 || (j0 % a.img_w) == a.img_w - 1;
    const bool g2z1 = !ok1 || (j1 % a.img_w) == a.img_w - 1;
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    unsigned long long *const mail = a.mail;
    const bool up = rank > 0, down = rank + 1 < G;

    float2 p1[NR], p2[NR], v[NR], c[NR], w[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int gi = r0 + r - 2;
        float2 x1 = make_float2(0.0f, 0.0f), x2 = x1, xv = x1;
        float2 xc = make_float2(INFINITY, INFINITY);
        if (gi >= -PAD_R && gi < H + PAD_R) {
            const int64_t o = (int64_t)gi * a.pitch;
            if (ok0) {
                x1.x = a.p1_in[o + swz(j0)];
                x2.x = a.p2_in[o + swz(j0)];
                xv.x = a.v_in[o + swz(j0)];
                xc.x = a.c[o + swz(j0)];
            }
            if (ok1) {
                x1.y = a.p1_in[o + swz(j1)];
                x2.y = a.p2_in[o + swz(j1)];
                xv.y = a.v_in[o + swz(j1)];
                xc.y = a.c[o + swz(j1)];
            }
        }
        p1[r] = x1;
        p2[r] = x2;
        v[r] = xv;
        c[r] = xc;
        w[r] = make_float2(0.0f, 0.0f);
    }
    const bool empty = a.n_rd != nullptr && *a.n_rd == 0;  // every pixel pinned: nothing moves
    const int K = empty ? 0 : a.K;
    if (lane == 31) {
#pragma unroll
        for (int r = 1; r < NR; ++r) eP[warp][r] = p2[r].y;
    }
    __syncthreads();

    // phase A at local row r: w = div rho - v / theta (rho2 of the left column: lane 0 takes
    // the previous warp's lane 31 from eP, or the given value for the halo row R)
    auto phaseA = [&](int r, float lhalo) {
        float l2 = __shfl_up_sync(FULL, p2[r].y, 1);
        if (lane == 0) l2 = warp == 0 ? 0.0f : (r == NR - 1 ? lhalo : eP[warp - 1][r]);
        const float d0 = __fadd_rn(__fsub_rn(p1[r].x, p1[r - 1].x), __fsub_rn(p2[r].x, l2));
        const float d1 = __fadd_rn(__fsub_rn(p1[r].y, p1[r - 1].y), __fsub_rn(p2[r].y, p2[r].x));
        w[r].x = __fmaf_rn(v[r].x, -inv_theta, d0);
        w[r].y = __fmaf_rn(v[r].y, -inv_theta, d1);
    };
    // phase B at local row r: rho' in place (w of the right column: lane 31 from eW)
    auto phaseB = [&](int r) {
        float wr = __shfl_down_sync(FULL, w[r].x, 1);
        if (lane == 31) wr = warp + 1 < NW ? eW[warp + 1][r] : 0.0f;
        const bool bottom = r0 + r - 2 == H - 1;
        {
            const float g1 = bottom ? 0.0f : __fsub_rn(w[r + 1].x, w[r].x);
            const float g2 = g2z0 ? 0.0f : __fsub_rn(w[r].y, w[r].x);
            const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(c[r].x)));
            const float rr = rcp_gx(__fmaf_rn(sqrt_gx(s), tau, 1.0f));
            p1[r].x = __fmul_rn(__fmaf_rn(g1, tau, p1[r].x), rr);
            p2[r].x = __fmul_rn(__fmaf_rn(g2, tau, p2[r].x), rr);
        }
        {
            const float g1 = bottom ? 0.0f : __fsub_rn(w[r + 1].y, w[r].y);
            const float g2 = g2z1 ? 0.0f : __fsub_rn(wr, w[r].y);
            const float s = __fmaf_rn(g1, g1, __fmaf_rn(g2, g2, fabsf(c[r].y)));
            const float rr = rcp_gx(__fmaf_rn(sqrt_gx(s), tau, 1.0f));
            p1[r].y = __fmul_rn(__fmaf_rn(g1, tau, p1[r].y), rr);
            p2[r].y = __fmul_rn(__fmaf_rn(g2, tau, p2[r].y), rr);
        }
    };
    // phase C at local row r: u, v' (u and the mask written out at the last iteration)
    auto phaseC = [&](int r, bool last) {
        float l2 = __shfl_up_sync(FULL, p2[r].y, 1);
        if (lane == 0) l2 = warp > 0 ? eP[warp - 1][r] : 0.0f;
        const float dn0 = __fadd_rn(__fsub_rn(p1[r].x, p1[r - 1].x), __fsub_rn(p2[r].x, l2));
        const float dn1 =
            __fadd_rn(__fsub_rn(p1[r].y, p1[r - 1].y), __fsub_rn(p2[r].y, p2[r].x));
        const float u0 = __fmaf_rn(dn0, -theta, v[r].x);
        const float u1 = __fmaf_rn(dn1, -theta, v[r].y);
        if (last) {
            const int gi = r0 + r - 2;
            if (gi < H) {
                const int64_t o = (int64_t)gi * a.pitch;
                const float ou0 = fabsf(c[r].x) < INFINITY ? u0 : v[r].x;
                const float ou1 = fabsf(c[r].y) < INFINITY ? u1 : v[r].y;
                if (ok0) {
                    a.u_out[o + j0] = ou0;
                    a.mask_out[o + j0] = ou0 > 0.5f;
                }
                if (ok1) {
                    a.u_out[o + j1] = ou1;
                    a.mask_out[o + j1] = ou1 > 0.5f;
                }
            }
        }
        v[r].x = __saturatef(__fmaf_rn(c[r].x, -0x1p100f, u0));
        v[r].y = __saturatef(__fmaf_rn(c[r].y, -0x1p100f, u1));
    };
    const int q = t;  // the thread's column pair (j0, j1) in a mailbox row
    auto slot = [&](int k, int g) { return mail + ((int64_t)(k & 1) * G + g) * 7 * NC; };

#ifdef RDS_GRID_PROFILE
    long long c_int = 0, c_wait = 0, c_bnd = 0, c_pub = 0, c_t0 = clock64();
#endif
    for (int k = 0; k < K; ++k) {
        const bool last = k + 1 == K;
#ifdef RDS_GRID_PROFILE
        long long c_a = clock64();
#endif
        // ---- interior rows: no halo needed
#pragma unroll
        for (int r = 3; r <= R + 1; ++r) phaseA(r, 0.0f);
        if (lane == 0) {
#pragma unroll
            for (int r = 3; r <= R + 1; ++r) eW[warp][r] = w[r].x;
        }
        __syncthreads();
#pragma unroll
        for (int r = 3; r <= R; ++r) phaseB(r);
        if (lane == 31) {
#pragma unroll
            for (int r = 3; r <= R; ++r) eP[warp][r] = p2[r].y;
        }
        __syncthreads();
#pragma unroll
        for (int r = 4; r <= R; ++r) phaseC(r, last);
        // ---- the neighbours' rows of iteration k - 1 (k = 0: the initial state, loaded)
        float lhalo = 0.0f;  // rho2 of row R in the column left of j0 (lane 0 of warps > 0)
#ifdef RDS_GRID_PROFILE
        long long c_b = clock64();
        c_int += c_b - c_a;
#endif
        if (k > 0) {
            // every word this thread needs is requested at once, then re-polled until all carry
            // the tag (one L2 round trip when they have already landed)
            const unsigned tag = a.tag0 + (unsigned)(k - 1);
            const unsigned long long *mu = slot(k - 1, rank - 1), *md = slot(k - 1, rank + 1);
            const bool edge_l = down && lane == 0 && warp > 0;
            unsigned long long x[15];
            unsigned long long spins = 0;
#ifndef RDS_GRID_ALLPOLL
            // one lane per warp polls one word per neighbour (the last row its writer warp
            // stores); the others wait at the warp barrier instead of flooding L2 with polls
            if (lane == 0) {
                if (up)
                    while (!ll_ok(ll_ld1(mu + 2 * (5 * NT + q)), tag)) {
                        RDS_GRID_BACKOFF;
                        if (++spins > (1ull << 31)) __trap();
                    }
                if (down)
                    while (!ll_ok(ll_ld1(md + 2 * (6 * NT + q)), tag)) {
                        RDS_GRID_BACKOFF;
                        if (++spins > (1ull << 31)) __trap();
                    }
            }
            __syncwarp();
#endif
            for (;;) {
                bool ok = true;
                if (up) {
                    ll_ld2(mu + 2 * (0 * NT + q), x[0], x[1]);
                    ll_ld2(mu + 2 * (1 * NT + q), x[2], x[3]);
                    ll_ld2(mu + 2 * (3 * NT + q), x[4], x[5]);
                    ll_ld2(mu + 2 * (5 * NT + q), x[6], x[7]);
#pragma unroll
                    for (int i = 0; i < 8; ++i) ok = ok && ll_ok(x[i], tag);
                }
                if (down) {
                    ll_ld2(md + 2 * (2 * NT + q), x[8], x[9]);
                    ll_ld2(md + 2 * (4 * NT + q), x[10], x[11]);
                    ll_ld2(md + 2 * (6 * NT + q), x[12], x[13]);
#pragma unroll
                    for (int i = 8; i < 14; ++i) ok = ok && ll_ok(x[i], tag);
                }
                if (edge_l) {
                    x[14] = ll_ld1(md + 4 * NC + j0 - 1);
                    ok = ok && ll_ok(x[14], tag);
                }
                if (ok) break;
                if (++spins > (1ull << 31)) __trap();  // cannot happen with co-resident CTAs
            }
            if (up) {
                p1[0] = make_float2(ll_val(x[0]), ll_val(x[1]));
                p1[1] = make_float2(ll_val(x[2]), ll_val(x[3]));
                p2[1] = make_float2(ll_val(x[4]), ll_val(x[5]));
                v[1] = make_float2(ll_val(x[6]), ll_val(x[7]));
            }
            if (down) {
                p1[NR - 1] = make_float2(ll_val(x[8]), ll_val(x[9]));
                p2[NR - 1] = make_float2(ll_val(x[10]), ll_val(x[11]));
                v[NR - 1] = make_float2(ll_val(x[12]), ll_val(x[13]));
            }
            if (edge_l) lhalo = ll_val(x[14]);
        } else if (lane == 0 && warp > 0) {
            lhalo = eP[warp - 1][NR - 1];  // the initial state's row R (written before the loop)
        }
#ifdef RDS_GRID_PROFILE
        long long c_c = clock64();
        c_wait += c_c - c_b;
#endif
        // ---- boundary rows
        phaseA(1, lhalo);
        phaseA(2, lhalo);
        phaseA(NR - 1, lhalo);
        if (lane == 0) {
            eW[warp][1] = w[1].x;
            eW[warp][2] = w[2].x;
            eW[warp][NR - 1] = w[NR - 1].x;
        }
        __syncthreads();
        phaseB(1);
        phaseB(2);
        phaseB(R + 1);
        if (lane == 31) {
            eP[warp][1] = p2[1].y;
            eP[warp][2] = p2[2].y;
            eP[warp][R + 1] = p2[R + 1].y;
        }
        __syncthreads();
        phaseC(2, last);
        if (R + 1 != 3) phaseC(3, last);
        phaseC(R + 1, last);
#ifdef RDS_GRID_PROFILE
        long long c_d = clock64();
        c_bnd += c_d - c_c;
#endif
        // ---- publish rows 0, R-2 (rho1), R-1 of iteration k
        {
            const unsigned tag = a.tag0 + (unsigned)k;
            unsigned long long *ms = slot(k, rank);
            ll_st2(ms + 2 * (0 * NT + q), p1[R], tag);
            ll_st2(ms + 2 * (1 * NT + q), p1[R + 1], tag);
            ll_st2(ms + 2 * (2 * NT + q), p1[2], tag);
            ll_st2(ms + 2 * (3 * NT + q), p2[R + 1], tag);
            ll_st2(ms + 2 * (4 * NT + q), p2[2], tag);
            ll_st2(ms + 2 * (5 * NT + q), v[R + 1], tag);
            ll_st2(ms + 2 * (6 * NT + q), v[2], tag);
        }
#ifdef RDS_GRID_PROFILE
        c_pub += clock64() - c_d;
#endif
    }
#ifdef RDS_GRID_PROFILE
    if ((t == 0 || t == NT - 1) && (rank % 37 == 0 || rank == G / 2))
        printf("grid prof rank %d t %d K %d: total %lld int %lld wait %lld bnd %lld pub %lld (cycles/iter)\n",
               rank, t, K, (clock64() - c_t0) / K, c_int / K, c_wait / K, c_bnd / K, c_pub / K);
#endif
    // The state is written back in place, over rows the neighbours read at the start.  K >= 2:
    // each neighbour has published (after a barrier that follows its initial loads); K = 1:
    // wait for its iteration-0 words here.
    if (K == 1) {
        const unsigned tag = a.tag0;
        if (up) (void)ll_wait2(slot(0, rank - 1) + 2 * q, tag);
        if (down) (void)ll_wait2(slot(0, rank + 1) + 2 * q, tag);
        __syncthreads();
    }
    // outputs: the state (u and the mask were written by the last iteration; K = 0: u0 = v)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int gi = r0 + r;
        if (gi >= H) break;
        const int64_t o = (int64_t)gi * a.pitch;
        if (K == 0) {
            if (ok0) {
                a.u_out[o + j0] = v[r + 2].x;
                a.mask_out[o + j0] = v[r + 2].x > 0.5f;
            }
            if (ok1) {
                a.u_out[o + j1] = v[r + 2].y;
                a.mask_out[o + j1] = v[r + 2].y > 0.5f;
            }
            continue;
        }
        if (ok0) {
            a.p1_out[o + swz(j0)] = p1[r + 2].x;
            a.p2_out[o + swz(j0)] = p2[r + 2].x;
            a.v_out[o + swz(j0)] = v[r + 2].x;
        }
        if (ok1) {
            a.p1_out[o + swz(j1)] = p1[r + 2].y;
            a.p2_out[o + swz(j1)] = p2[r + 2].y;
            a.v_out[o + swz(j1)] = v[r + 2].y;
        }
    }
}

typedef void (*GridFn)(const GridArgs);
static GridFn grid_fn(int R) {
    switch (R) {
        case 2: return k_grid<2>;
        case 3: return k_grid<3>;
        case 4: return k_grid<4>;
        case 5: return k_grid<5>;
        case 6: return k_grid<6>;
        case 7: return k_grid<7>;
        case 8: return k_grid<8>;
        default: return nullptr;
    }
}

static int grid_threads(int W) { return (W + 63) / 64 * 32; }

// Slabs for an H x W image on n_sm SMs: the smallest R in 2 .. 8 with G = ceil(H / R) <= n_sm
// co-resident CTAs (one per SM), two columns per thread (W <= 1024).
bool grid_plan(int64_t H, int64_t W, int n_sm, int *G_out, int *R_out) {
    if (H < 1 || W < 1 || W > 2 * GRID_THREADS) return false;
    for (int R = 2; R <= 8; ++R) {
        const int64_t G = (H + R - 1) / R;
        if (G <= n_sm) {
            *G_out = (int)G;
            *R_out = R;
            return true;
        }
    }
    return false;
}

size_t grid_mail_words(int G, int W) { return (size_t)2 * G * 7 * 2 * grid_threads(W); }

// Can G CTAs of this shape be co-resident here (cooperative launch)?
bool grid_fits(const GridArgs &a) {
    GridFn fn = grid_fn(a.R);
    if (!fn) return false;
    int per_sm = 0, dev = 0, n_sm = 0;
    bool ok = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)fn,
                                                            grid_threads(a.W), 0) == cudaSuccess &&
              cudaGetDevice(&dev) == cudaSuccess &&
              cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess;
    ok = ok && (int64_t)per_sm * n_sm >= a.G;
    (void)cudaGetLastError();
    return ok;
}

cudaError_t launch_grid(const GridArgs &a, cudaStream_t s) {
    GridFn fn = grid_fn(a.R);
    if (!fn) return cudaErrorInvalidValue;
    void *args[] = {const_cast<GridArgs *>(&a)};
    return cudaLaunchCooperativeKernel((const void *)fn, dim3(a.G), dim3(grid_threads(a.W)),
                                       args, 0, s);
}

}  // namespace rds
