// k_vol.cu -- f4: the restricted-domain dual iteration on 3-D volumes (§5
// "extension to 3D"), sm_100a.  Same method as the 2-D path, operators extended axis by axis
// (reading R-F4): grad = forward differences along i (rows), j (columns), k (planes) with a
// zero last row / column / plane, div = -grad^T, rho = (rho1, rho2, rho3).
//
// Layout: padded volume, voxel (k, i, j) at origin + k * plane + i * pitch + j with 2 frame
// planes before and after, 2 frame rows above and 32 below, 4 frame columns left and >= 32
// right (a CTA window reaches 2 before its tile and up to VT_Y / 32 past the last image
// row / column); the frame holds pinned background (rho = 0, v = 0, c' = +inf), so no load
// is bounds-checked.  c' = 2^-100 theta*lambda*f on RD, -inf on Fg, +inf on Bg (as in 2-D).
//
// k_vol_step: one iteration per launch, all of it in one pass over the volume (36 B per
// voxel: read rho1..3, v, c'; write rho1..3, v).  A CTA of 32 x 16 threads owns one (i, j)
// column each of a 16 x 32 window and marches along k through a z-chunk: per plane step n it
// loads plane n, forms w(n) = div rho(n) - v(n)/theta, the rho update of plane n-1 (needs
// w(n-1), w(n)), and the u- and v-steps of plane n-1 (need rho_new of plane n-1 at i-1, j-1
// and of plane n-2).  Windows overlap by 3 columns / rows (the dependency cone of one
// iteration), so each CTA writes a 13 x 29 tile; three __syncthreads per plane step.
#include <math.h>
#include <stdlib.h>

#include "internal.h"

namespace rds {

#ifndef RDS_VOL_TY
#define RDS_VOL_TY 16
#endif
constexpr int VT_X = 32, VT_Y = RDS_VOL_TY;  // threads per CTA (columns, rows)
constexpr int VO_X = VT_X - 3, VO_Y = VT_Y - 3;  // output tile (29 x 13)

__device__ __forceinline__ float vsqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float vrcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <bool WRITE_U>
__global__ void __launch_bounds__(VT_X * VT_Y) k_vol_step(const VolArgs a) {
    __shared__ float s1[VT_Y][VT_X], s2[VT_Y][VT_X];   // rho1, rho2 of plane n
    __shared__ float sw[2][VT_Y][VT_X];                // w of planes n-1, n (alternating)
    __shared__ float q1s[VT_Y][VT_X], q2s[VT_Y][VT_X]; // rho1, rho2 new of plane n-1
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int j = blockIdx.x * VO_X - 2 + tx, i = blockIdx.y * VO_Y - 2 + ty;
    const int k0 = blockIdx.z * a.kz, k1 = min(k0 + a.kz, a.D);
    // every thread owns a column inside the padded frame (the frame is >= 2 wide)
    const int64_t col = (int64_t)i * a.pitch + j;
    const bool in_w = ty >= 1 && tx >= 1;                          // w needed here
    const bool in_q = ty >= 1 && ty <= VT_Y - 2 && tx >= 1 && tx <= VT_X - 2;  // rho_new
    const bool in_o = ty >= 2 && ty <= VT_Y - 2 && tx >= 2 && tx <= VT_X - 2 && i < a.H &&
                      j < a.W;                                     // u, v output
    const bool last_i = i == a.H - 1, last_j = j == a.W - 1;
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    // pipeline registers: plane n-1 values of this column
    // (the first step's plane n-1 = k0-2 only feeds w(k0-1) through rho3; its other values
    // feed results that are discarded)
    float pp1 = 0.f, pp2 = 0.f, pv = 0.f, pc = INFINITY;           // old rho, v, c' at n-1
    float pp3 = a.p3_in[(int64_t)(k0 - 2) * a.plane + col];
    float q3prev = 0.f;                                            // rho3 new at plane n-2
    int cur = 0;
    // plane n+1 is loaded one step ahead (registers), so HBM latency hides behind a step
    int64_t o_next = (int64_t)(k0 - 1) * a.plane + col;
    float x1 = a.p1_in[o_next], x2 = a.p2_in[o_next], x3 = a.p3_in[o_next];
    float xv = a.v_in[o_next], xc = a.c[o_next];
    for (int n = k0 - 1; n <= k1; ++n) {
        const float p1n = x1, p2n = x2, p3n = x3, vn = xv, cn = xc;
        if (n < k1) {
            o_next += a.plane;
            x1 = a.p1_in[o_next];
            x2 = a.p2_in[o_next];
            x3 = a.p3_in[o_next];
            xv = a.v_in[o_next];
            xc = a.c[o_next];
        }
        s1[ty][tx] = p1n;
        s2[ty][tx] = p2n;
        __syncthreads();
        // w(n) = div rho(n) - v(n)/theta; the p3 of plane n-1 is pp3 (this column)
        float wn = 0.f;
        if (in_w) {
            const float d = (p1n - s1[ty - 1][tx]) + (p2n - s2[ty][tx - 1]) + (p3n - pp3);
            wn = fmaf(vn, -inv_theta, d);
        }
        sw[cur][ty][tx] = wn;
        __syncthreads();
        // rho-step at plane n-1 (Eq. 8): g from w(n-1) (sw[cur^1]) and w(n)
        float q1 = 0.f, q2 = 0.f, q3 = 0.f;
        if (in_q) {
            const float w0 = sw[cur ^ 1][ty][tx];
            const float g1 = last_i ? 0.f : sw[cur ^ 1][ty + 1][tx] - w0;
            const float g2 = last_j ? 0.f : sw[cur ^ 1][ty][tx + 1] - w0;
            const float g3 = (n - 1 == a.D - 1) ? 0.f : wn - w0;
            const float s = fmaf(g1, g1, fmaf(g2, g2, fmaf(g3, g3, fabsf(pc))));
            const float rr = vrcp(fmaf(tau, vsqrt(s), 1.0f));
            q1 = fmaf(tau, g1, pp1) * rr;
            q2 = fmaf(tau, g2, pp2) * rr;
            q3 = fmaf(tau, g3, pp3) * rr;
        }
        q1s[ty][tx] = q1;
        q2s[ty][tx] = q2;
        __syncthreads();
        // u- and v-steps at plane n-1 (Eq. 7, 9), output planes [k0, k1)
        if (in_o && n - 1 >= k0) {
            const float d = (q1 - q1s[ty - 1][tx]) + (q2 - q2s[ty][tx - 1]) + (q3 - q3prev);
            const float u = fmaf(-theta, d, pv);
            const float vnew = __saturatef(fmaf(pc, -0x1p100f, u));
            const int64_t oo = (int64_t)(n - 1) * a.plane + col;
            a.p1_out[oo] = q1;
            a.p2_out[oo] = q2;
            a.p3_out[oo] = q3;
            a.v_out[oo] = vnew;
            if (WRITE_U) {
                const float uu = fabsf(pc) < INFINITY ? u : pv;  // pinned u0 off RD
                a.u_out[oo] = uu;
                a.mask_out[oo] = uu > 0.5f;
            }
        }
        // rotate the pipeline
        pp1 = p1n;
        pp2 = p2n;
        pp3 = p3n;
        pv = vn;
        pc = cn;
        q3prev = q3;
        cur ^= 1;
    }
}

// Two rows per thread (round 2): a CTA of 32 x 8 threads covers the same 32 x 16 window, each
// thread the rows i = 2 ty and 2 ty + 1 of its column, so the three __syncthreads of a plane
// step are paid for twice the work and half of the row neighbours (rho1 at i - 1, w at i + 1,
// rho1' at i - 1) come from the thread's own registers.  The same float operations in the same
// order as k_vol_step (results bit-identical).
constexpr int VT2_Y = VT_Y / 2;  // thread rows

template <bool WRITE_U>
__global__ void __launch_bounds__(VT_X * VT2_Y) k_vol_step2(const VolArgs a) {
    __shared__ float s1[VT_Y][VT_X], s2[VT_Y][VT_X];   // rho1, rho2 of plane n
    __shared__ float sw[2][VT_Y][VT_X];                // w of planes n-1, n (alternating)
    __shared__ float q1s[VT_Y][VT_X], q2s[VT_Y][VT_X]; // rho1, rho2 new of plane n-1
    const int tx = threadIdx.x, ty0 = 2 * threadIdx.y;  // local rows ty0, ty0 + 1
    const int j = blockIdx.x * VO_X - 2 + tx, i0 = blockIdx.y * VO_Y - 2 + ty0;
    const int k0 = blockIdx.z * a.kz, k1 = min(k0 + a.kz, a.D);
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    bool in_w[2], in_q[2], in_o[2], last_i[2];
    int64_t col[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int ty = ty0 + r, i = i0 + r;
        col[r] = (int64_t)i * a.pitch + j;
        in_w[r] = ty >= 1 && tx >= 1;
        in_q[r] = ty >= 1 && ty <= VT_Y - 2 && tx >= 1 && tx <= VT_X - 2;
        in_o[r] = ty >= 2 && ty <= VT_Y - 2 && tx >= 2 && tx <= VT_X - 2 && i < a.H && j < a.W;
        last_i[r] = i == a.H - 1;
    }
    const bool last_j = j == a.W - 1;
    float pp1[2] = {0.f, 0.f}, pp2[2] = {0.f, 0.f}, pv[2] = {0.f, 0.f};
    float pc[2] = {INFINITY, INFINITY}, q3prev[2] = {0.f, 0.f}, pp3[2];
    float x1[2], x2[2], x3[2], xv[2], xc[2];
    int64_t o_next[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        pp3[r] = a.p3_in[(int64_t)(k0 - 2) * a.plane + col[r]];
        o_next[r] = (int64_t)(k0 - 1) * a.plane + col[r];
        x1[r] = a.p1_in[o_next[r]];
        x2[r] = a.p2_in[o_next[r]];
        x3[r] = a.p3_in[o_next[r]];
        xv[r] = a.v_in[o_next[r]];
        xc[r] = a.c[o_next[r]];
    }
    int cur = 0;
    for (int n = k0 - 1; n <= k1; ++n) {
        float p1n[2], p2n[2], p3n[2], vn[2], cn[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            p1n[r] = x1[r];
            p2n[r] = x2[r];
            p3n[r] = x3[r];
            vn[r] = xv[r];
            cn[r] = xc[r];
            if (n < k1) {
                o_next[r] += a.plane;
                x1[r] = a.p1_in[o_next[r]];
                x2[r] = a.p2_in[o_next[r]];
                x3[r] = a.p3_in[o_next[r]];
                xv[r] = a.v_in[o_next[r]];
                xc[r] = a.c[o_next[r]];
            }
            s1[ty0 + r][tx] = p1n[r];
            s2[ty0 + r][tx] = p2n[r];
        }
        __syncthreads();
        float wn[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ty = ty0 + r;
            wn[r] = 0.f;
            if (in_w[r]) {
                const float up1 = r == 1 ? p1n[0] : s1[ty - 1][tx];
                const float d = (p1n[r] - up1) + (p2n[r] - s2[ty][tx - 1]) + (p3n[r] - pp3[r]);
                wn[r] = fmaf(vn[r], -inv_theta, d);
            }
            sw[cur][ty][tx] = wn[r];
        }
        __syncthreads();
        float q1[2], q2[2], q3[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ty = ty0 + r;
            q1[r] = q2[r] = q3[r] = 0.f;
            if (in_q[r]) {
                const float w0 = sw[cur ^ 1][ty][tx];
                const float g1 = last_i[r] ? 0.f : sw[cur ^ 1][ty + 1][tx] - w0;
                const float g2 = last_j ? 0.f : sw[cur ^ 1][ty][tx + 1] - w0;
                const float g3 = (n - 1 == a.D - 1) ? 0.f : wn[r] - w0;
                const float s = fmaf(g1, g1, fmaf(g2, g2, fmaf(g3, g3, fabsf(pc[r]))));
                const float rr = vrcp(fmaf(tau, vsqrt(s), 1.0f));
                q1[r] = fmaf(tau, g1, pp1[r]) * rr;
                q2[r] = fmaf(tau, g2, pp2[r]) * rr;
                q3[r] = fmaf(tau, g3, pp3[r]) * rr;
            }
            q1s[ty][tx] = q1[r];
            q2s[ty][tx] = q2[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ty = ty0 + r;
            if (in_o[r] && n - 1 >= k0) {
                const float qup = r == 1 ? q1[0] : q1s[ty - 1][tx];
                const float d = (q1[r] - qup) + (q2[r] - q2s[ty][tx - 1]) + (q3[r] - q3prev[r]);
                const float u = fmaf(-theta, d, pv[r]);
                const float vnew = __saturatef(fmaf(pc[r], -0x1p100f, u));
                const int64_t oo = (int64_t)(n - 1) * a.plane + col[r];
                a.p1_out[oo] = q1[r];
                a.p2_out[oo] = q2[r];
                a.p3_out[oo] = q3[r];
                a.v_out[oo] = vnew;
                if (WRITE_U) {
                    const float uu = fabsf(pc[r]) < INFINITY ? u : pv[r];
                    a.u_out[oo] = uu;
                    a.mask_out[oo] = uu > 0.5f;
                }
            }
            pp1[r] = p1n[r];
            pp2[r] = p2n[r];
            pp3[r] = p3n[r];
            pv[r] = vn[r];
            pc[r] = cn[r];
            q3prev[r] = q3[r];
        }
        cur ^= 1;
    }
}

// Two barriers per plane step (RDS_VOL_2BAR): rho1 / rho2 of plane n + 1 go into the other of
// two shared slots during step n's rho phase, so the barrier that publishes the new rho also
// publishes them and the next step's w phase needs no barrier of its own.  Same operations.
template <bool WRITE_U>
__global__ void __launch_bounds__(VT_X * VT2_Y) k_vol_step2b(const VolArgs a) {
    __shared__ float s1[2][VT_Y][VT_X], s2[2][VT_Y][VT_X];  // rho1, rho2 of planes n, n+1
    __shared__ float sw[2][VT_Y][VT_X];                // w of planes n-1, n (alternating)
    __shared__ float q1s[VT_Y][VT_X], q2s[VT_Y][VT_X]; // rho1, rho2 new of plane n-1
    const int tx = threadIdx.x, ty0 = 2 * threadIdx.y;  // local rows ty0, ty0 + 1
    const int j = blockIdx.x * VO_X - 2 + tx, i0 = blockIdx.y * VO_Y - 2 + ty0;
    const int k0 = blockIdx.z * a.kz, k1 = min(k0 + a.kz, a.D);
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    bool in_w[2], in_q[2], in_o[2], last_i[2];
    int64_t col[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int ty = ty0 + r, i = i0 + r;
        col[r] = (int64_t)i * a.pitch + j;
        in_w[r] = ty >= 1 && tx >= 1;
        in_q[r] = ty >= 1 && ty <= VT_Y - 2 && tx >= 1 && tx <= VT_X - 2;
        in_o[r] = ty >= 2 && ty <= VT_Y - 2 && tx >= 2 && tx <= VT_X - 2 && i < a.H && j < a.W;
        last_i[r] = i == a.H - 1;
    }
    const bool last_j = j == a.W - 1;
    float pp1[2] = {0.f, 0.f}, pp2[2] = {0.f, 0.f}, pv[2] = {0.f, 0.f};
    float pc[2] = {INFINITY, INFINITY}, q3prev[2] = {0.f, 0.f}, pp3[2];
    float x1[2], x2[2], x3[2], xv[2], xc[2];
    int64_t o_next[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        pp3[r] = a.p3_in[(int64_t)(k0 - 2) * a.plane + col[r]];
        o_next[r] = (int64_t)(k0 - 1) * a.plane + col[r];
        x1[r] = a.p1_in[o_next[r]];
        x2[r] = a.p2_in[o_next[r]];
        x3[r] = a.p3_in[o_next[r]];
        xv[r] = a.v_in[o_next[r]];
        xc[r] = a.c[o_next[r]];
    }
    // plane k0 - 1 into its rho1 / rho2 slot (the loop stores plane n + 1 during step n)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        s1[(k0 - 1) & 1][ty0 + r][tx] = x1[r];
        s2[(k0 - 1) & 1][ty0 + r][tx] = x2[r];
    }
    __syncthreads();
    int cur = 0;
    for (int n = k0 - 1; n <= k1; ++n) {
        const int sb = n & 1;
        float p1n[2], p2n[2], p3n[2], vn[2], cn[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            p1n[r] = x1[r];
            p2n[r] = x2[r];
            p3n[r] = x3[r];
            vn[r] = xv[r];
            cn[r] = xc[r];
            if (n < k1) {
                o_next[r] += a.plane;
                x1[r] = a.p1_in[o_next[r]];
                x2[r] = a.p2_in[o_next[r]];
                x3[r] = a.p3_in[o_next[r]];
                xv[r] = a.v_in[o_next[r]];
                xc[r] = a.c[o_next[r]];
            }
        }
        float wn[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ty = ty0 + r;
            wn[r] = 0.f;
            if (in_w[r]) {
                const float up1 = r == 1 ? p1n[0] : s1[sb][ty - 1][tx];
                const float d =
                    (p1n[r] - up1) + (p2n[r] - s2[sb][ty][tx - 1]) + (p3n[r] - pp3[r]);
                wn[r] = fmaf(vn[r], -inv_theta, d);
            }
            sw[cur][ty][tx] = wn[r];
        }
        __syncthreads();
        float q1[2], q2[2], q3[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ty = ty0 + r;
            q1[r] = q2[r] = q3[r] = 0.f;
            if (in_q[r]) {
                const float w0 = sw[cur ^ 1][ty][tx];
                const float g1 = last_i[r] ? 0.f : sw[cur ^ 1][ty + 1][tx] - w0;
                const float g2 = last_j ? 0.f : sw[cur ^ 1][ty][tx + 1] - w0;
                const float g3 = (n - 1 == a.D - 1) ? 0.f : wn[r] - w0;
                const float s = fmaf(g1, g1, fmaf(g2, g2, fmaf(g3, g3, fabsf(pc[r]))));
                const float rr = vrcp(fmaf(tau, vsqrt(s), 1.0f));
                q1[r] = fmaf(tau, g1, pp1[r]) * rr;
                q2[r] = fmaf(tau, g2, pp2[r]) * rr;
                q3[r] = fmaf(tau, g3, pp3[r]) * rr;
            }
            q1s[ty][tx] = q1[r];
            q2s[ty][tx] = q2[r];
            // plane n + 1 (prefetched at the top of this step) into the other slot: the
            // barrier below also publishes it for the next step's w
            s1[sb ^ 1][ty][tx] = x1[r];
            s2[sb ^ 1][ty][tx] = x2[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ty = ty0 + r;
            if (in_o[r] && n - 1 >= k0) {
                const float qup = r == 1 ? q1[0] : q1s[ty - 1][tx];
                const float d = (q1[r] - qup) + (q2[r] - q2s[ty][tx - 1]) + (q3[r] - q3prev[r]);
                const float u = fmaf(-theta, d, pv[r]);
                const float vnew = __saturatef(fmaf(pc[r], -0x1p100f, u));
                const int64_t oo = (int64_t)(n - 1) * a.plane + col[r];
                a.p1_out[oo] = q1[r];
                a.p2_out[oo] = q2[r];
                a.p3_out[oo] = q3[r];
                a.v_out[oo] = vnew;
                if (WRITE_U) {
                    const float uu = fabsf(pc[r]) < INFINITY ? u : pv[r];
                    a.u_out[oo] = uu;
                    a.mask_out[oo] = uu > 0.5f;
                }
            }
            pp1[r] = p1n[r];
            pp2[r] = p2n[r];
            pp3[r] = p3n[r];
            pv[r] = vn[r];
            pc[r] = cn[r];
            q3prev[r] = q3[r];
        }
        cur ^= 1;
    }
}

// ---------------------------------------------------------------------------------------
// k_vol_tb<S>: S iterations per pass over the volume (temporal blocking along the plane
// axis).  The S stages of a CTA are a software pipeline: at plane step n stage s takes the
// state of level s at plane n - 2s (stage 0 from HBM, stage s > 0 from the registers stage s-1
// filled at step n - 1), runs the three phases of k_vol_step2 on it (w of that plane, the rho
// update of the plane before it, the u- and v-steps of that plane) and hands the new level-
// (s+1) state of plane n - 2s - 1 to stage s+1; the last stage writes it out.  All stages share
// the phase barriers (three per plane step).  A window of 32 x TY columns loses 2 rows /
// columns on its low side and 1 on its high side per stage (the dependency cone), so it writes
// a (32 - 3S) x (TY - 3S) tile; along the planes stage s produces valid state from plane
// k0 - S + s + 1 on, so the pass starts S planes before its z-chunk and reads up to S - 1
// planes past it (the frame, VOL_PZ >= S + 1).  Every float operation is k_vol_step's in the
// same order: S passes of k_vol_tb<1-stage> == S launches of k_vol_step, bit for bit (tested).
// ---------------------------------------------------------------------------------------
template <int S, int TY, bool WRITE_U>
#ifndef RDS_VTB_MINB
#define RDS_VTB_MINB 1
#endif
__global__ void __launch_bounds__(VT_X * TY / 2, RDS_VTB_MINB) k_vol_tb(const VolArgs a) {
    extern __shared__ float vsm[];
    constexpr int PL = TY * VT_X;           // one window plane
    constexpr int OX = VT_X - 3 * S, OY = TY - 3 * S;
    // per stage: s1, s2 (rho1, rho2 of its plane), sw[2] (w of its plane and the one before),
    // q1s, q2s (new rho1, rho2 of the plane before)
    auto S1 = [&](int st) { return vsm + (st * 6 + 0) * PL; };
    auto S2 = [&](int st) { return vsm + (st * 6 + 1) * PL; };
    auto SW = [&](int st, int c) { return vsm + (st * 6 + 2 + c) * PL; };
    auto Q1 = [&](int st) { return vsm + (st * 6 + 4) * PL; };
    auto Q2 = [&](int st) { return vsm + (st * 6 + 5) * PL; };
    const int tx = threadIdx.x, ty0 = 2 * threadIdx.y;  // local rows ty0, ty0 + 1
    const int j = blockIdx.x * OX - 2 * S + tx, i0 = blockIdx.y * OY - 2 * S + ty0;
    const int k0 = blockIdx.z * a.kz, k1 = min(k0 + a.kz, a.D);
    const float tau = a.tau, theta = a.theta, inv_theta = a.inv_theta;
    bool in_w[2], in_q[2], in_o[2], last_i[2];
    int64_t col[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int ty = ty0 + r, i = i0 + r;
        col[r] = (int64_t)i * a.pitch + j;
        in_w[r] = ty >= 1 && tx >= 1;
        in_q[r] = ty >= 1 && ty <= TY - 2 && tx >= 1 && tx <= VT_X - 2;
        in_o[r] = ty >= 2 * S && ty <= TY - 1 - S && tx >= 2 * S && tx <= VT_X - 1 - S &&
                  i < a.H && j < a.W;
        last_i[r] = i == a.H - 1;
    }
    const bool last_j = j == a.W - 1;
    // per stage and row: the state of the plane before the stage's current one (pp*, pv, pc),
    // rho3 new of the plane before that (q3prev), and the stage's output of the last step
    float pp1[S][2], pp2[S][2], pp3[S][2], pv[S][2], pc[S][2], q3prev[S][2];
    float o1[S][2], o2[S][2], o3[S][2], ov[S][2], oc[S][2];
#pragma unroll
    for (int st = 0; st < S; ++st)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            pp1[st][r] = pp2[st][r] = pp3[st][r] = pv[st][r] = q3prev[st][r] = 0.f;
            pc[st][r] = INFINITY;
            o1[st][r] = o2[st][r] = o3[st][r] = ov[st][r] = 0.f;
            oc[st][r] = INFINITY;
        }
    // stage 0 reads planes n0 .. nl (one ahead, in registers); planes past nl are not needed
    // by any valid output and read as the pinned frame
    const int n0 = k0 - S - 1, nl = k1 + S - 1, n1 = k1 + 2 * S - 2;
    float x1[2], x2[2], x3[2], xv[2], xc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int64_t o = (int64_t)n0 * a.plane + col[r];
        x1[r] = a.p1_in[o];
        x2[r] = a.p2_in[o];
        x3[r] = a.p3_in[o];
        xv[r] = a.v_in[o];
        xc[r] = a.c[o];
    }
    int cur = 0;
    for (int n = n0; n <= n1; ++n) {
        // L: each stage's current plane (stage 0: HBM; stage s: stage s-1's last output)
        float p1n[S][2], p2n[S][2], p3n[S][2], vn[S][2], cn[S][2];
#pragma unroll
        for (int st = S - 1; st >= 0; --st)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (st == 0) {
                    p1n[0][r] = x1[r];
                    p2n[0][r] = x2[r];
                    p3n[0][r] = x3[r];
                    vn[0][r] = xv[r];
                    cn[0][r] = xc[r];
                    if (n < nl) {
                        const int64_t o = (int64_t)(n + 1) * a.plane + col[r];
                        x1[r] = a.p1_in[o];
                        x2[r] = a.p2_in[o];
                        x3[r] = a.p3_in[o];
                        xv[r] = a.v_in[o];
                        xc[r] = a.c[o];
                    } else {
                        x1[r] = x2[r] = x3[r] = xv[r] = 0.f;
                        xc[r] = INFINITY;
                    }
                } else {
                    p1n[st][r] = o1[st - 1][r];
                    p2n[st][r] = o2[st - 1][r];
                    p3n[st][r] = o3[st - 1][r];
                    vn[st][r] = ov[st - 1][r];
                    cn[st][r] = oc[st - 1][r];
                }
                S1(st)[(ty0 + r) * VT_X + tx] = p1n[st][r];
                S2(st)[(ty0 + r) * VT_X + tx] = p2n[st][r];
            }
        __syncthreads();
        // W: w of each stage's current plane
        float wn[S][2];
#pragma unroll
        for (int st = 0; st < S; ++st)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ty = ty0 + r;
                wn[st][r] = 0.f;
                if (in_w[r]) {
                    const float up1 = r == 1 ? p1n[st][0] : S1(st)[(ty - 1) * VT_X + tx];
                    const float d = (p1n[st][r] - up1) + (p2n[st][r] - S2(st)[ty * VT_X + tx - 1]) +
                                    (p3n[st][r] - pp3[st][r]);
                    wn[st][r] = fmaf(vn[st][r], -inv_theta, d);
                }
                SW(st, cur)[ty * VT_X + tx] = wn[st][r];
            }
        __syncthreads();
        // Q: the rho update of each stage's plane before (its plane index m - 1, m = n - 2 st)
        float q1[S][2], q2[S][2], q3[S][2];
#pragma unroll
        for (int st = 0; st < S; ++st) {
            const bool last_k = n - 2 * st - 1 == a.D - 1;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ty = ty0 + r;
                q1[st][r] = q2[st][r] = q3[st][r] = 0.f;
                if (in_q[r]) {
                    const float *sw = SW(st, cur ^ 1);
                    const float w0 = sw[ty * VT_X + tx];
                    const float g1 = last_i[r] ? 0.f : sw[(ty + 1) * VT_X + tx] - w0;
                    const float g2 = last_j ? 0.f : sw[ty * VT_X + tx + 1] - w0;
                    const float g3 = last_k ? 0.f : wn[st][r] - w0;
                    const float s_ = fmaf(g1, g1, fmaf(g2, g2, fmaf(g3, g3, fabsf(pc[st][r]))));
                    const float rr = vrcp(fmaf(tau, vsqrt(s_), 1.0f));
                    q1[st][r] = fmaf(tau, g1, pp1[st][r]) * rr;
                    q2[st][r] = fmaf(tau, g2, pp2[st][r]) * rr;
                    q3[st][r] = fmaf(tau, g3, pp3[st][r]) * rr;
                }
                Q1(st)[ty * VT_X + tx] = q1[st][r];
                Q2(st)[ty * VT_X + tx] = q2[st][r];
            }
        }
        __syncthreads();
        // O: u, v' of each stage's plane before; the new state goes to the next stage (or out)
#pragma unroll
        for (int st = 0; st < S; ++st) {
            const int m = n - 2 * st - 1;  // the plane this stage finishes
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ty = ty0 + r;
                float vnew = 0.f, u = 0.f;
                if (in_w[r]) {
                    const float qup = r == 1 ? q1[st][0] : Q1(st)[(ty - 1) * VT_X + tx];
                    const float d = (q1[st][r] - qup) + (q2[st][r] - Q2(st)[ty * VT_X + tx - 1]) +
                                    (q3[st][r] - q3prev[st][r]);
                    u = fmaf(-theta, d, pv[st][r]);
                    vnew = __saturatef(fmaf(pc[st][r], -0x1p100f, u));
                }
                if (st == S - 1) {
                    if (in_o[r] && m >= k0 && m < k1) {
                        const int64_t oo = (int64_t)m * a.plane + col[r];
                        a.p1_out[oo] = q1[st][r];
                        a.p2_out[oo] = q2[st][r];
                        a.p3_out[oo] = q3[st][r];
                        a.v_out[oo] = vnew;
                        if (WRITE_U) {
                            const float uu = fabsf(pc[st][r]) < INFINITY ? u : pv[st][r];
                            a.u_out[oo] = uu;
                            a.mask_out[oo] = uu > 0.5f;
                        }
                    }
                } else {
                    o1[st][r] = q1[st][r];
                    o2[st][r] = q2[st][r];
                    o3[st][r] = q3[st][r];
                    ov[st][r] = vnew;
                    oc[st][r] = pc[st][r];
                }
                pp1[st][r] = p1n[st][r];
                pp2[st][r] = p2n[st][r];
                pp3[st][r] = p3n[st][r];
                pv[st][r] = vn[st][r];
                pc[st][r] = cn[st][r];
                q3prev[st][r] = q3[st][r];
            }
        }
        cur ^= 1;
    }
}

#ifndef RDS_VTB_TY
#define RDS_VTB_TY 32
#endif
constexpr int VTB_TY = RDS_VTB_TY;  // window rows of k_vol_tb (32 x 32 columns, 512 threads)

static size_t vol_tb_smem(int S) { return sizeof(float) * 6 * (size_t)S * VTB_TY * VT_X; }

template <int S>
static cudaError_t launch_tb(const VolArgs &a, bool write_u, cudaStream_t s) {
    constexpr int OX = VT_X - 3 * S, OY = VTB_TY - 3 * S;
    dim3 grid((a.W + OX - 1) / OX, (a.H + OY - 1) / OY, (a.D + a.kz - 1) / a.kz);
    dim3 block(VT_X, VTB_TY / 2);
    const size_t sm = vol_tb_smem(S);
    auto fn = write_u ? k_vol_tb<S, VTB_TY, true> : k_vol_tb<S, VTB_TY, false>;
    cudaError_t e = cudaFuncSetAttribute((const void *)fn,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    fn<<<grid, block, sm, s>>>(a);
    return cudaGetLastError();
}

int64_t vol_tb_tiles(int S, int64_t H, int64_t W) {
    const int OX = VT_X - 3 * S, OY = VTB_TY - 3 * S;
    return ((W + OX - 1) / OX) * ((H + OY - 1) / OY);
}

int vol_tb_blocks_per_sm(int S) {
    static int cache[VOL_TB_MAX + 1] = {0};
    if (S < 1 || S > VOL_TB_MAX) return 0;
    if (cache[S] == 0) {
        const void *fn = S == 1   ? (const void *)k_vol_tb<1, VTB_TY, false>
                         : S == 2 ? (const void *)k_vol_tb<2, VTB_TY, false>
                                  : (const void *)k_vol_tb<3, VTB_TY, false>;
        int b = 0;
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)vol_tb_smem(S)) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, VT_X * VTB_TY / 2,
                                                          vol_tb_smem(S)) != cudaSuccess ||
            b < 1)
            b = 1;
        (void)cudaGetLastError();
        cache[S] = b;
    }
    return cache[S];
}

cudaError_t launch_vol_tb(const VolArgs &a, int S, bool write_u, cudaStream_t s) {
    switch (S) {
        case 1: return launch_tb<1>(a, write_u, s);
        case 2: return launch_tb<2>(a, write_u, s);
        case 3: return launch_tb<3>(a, write_u, s);
        default: return cudaErrorInvalidValue;
    }
}

// K1 of the volume path: f (R-A1 order), label, c', u0 / mask, v0 and rho0 = 0 into both
// buffers; frame voxels are never touched (they keep the allocation-time pinned values).
__global__ void k_vol_setup(const VolSetupArgs a) {
    const int64_t n = (int64_t)a.D * a.H * a.W;
    const bool use_p = a.P != nullptr && a.gamma != 0.0f;
    unsigned long long n_rd = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = x / ((int64_t)a.H * a.W), r = x - k * a.H * a.W;
        const int i = (int)(r / a.W), j = (int)(r - (int64_t)i * a.W);
        const int64_t o = k * a.plane + (int64_t)i * a.pitch + j;
        const float z = a.z[o];
        const float aa = __fsub_rn(z, a.c1), bb = __fsub_rn(z, a.c2);
        float f = __fsub_rn(__fmul_rn(aa, aa), __fmul_rn(bb, bb));
        if (use_p) f = __fadd_rn(f, __fmul_rn(a.gamma, a.P[o]));
        const bool rd = fabsf(f) < a.delta, fg = f <= 0.0f;
        const float u0 = fg ? 1.0f : 0.0f;
        a.f[o] = f;
        a.lab[o] = rd ? 2 : (fg ? 1 : 0);
        a.c[o] = rd ? __fmul_rn(fminf(fmaxf(__fmul_rn(a.theta_lambda, f), -0x1p20f), 0x1p20f),
                                0x1p-100f)
                    : (fg ? -INFINITY : INFINITY);
        a.u[o] = u0;
        a.mask[o] = fg ? 1 : 0;
        a.v0[o] = a.v1[o] = u0;
        a.p10[o] = a.p11[o] = a.p20[o] = a.p21[o] = a.p30[o] = a.p31[o] = 0.0f;
        n_rd += rd;
    }
    if (n_rd) atomicAdd(a.n_rd, n_rd);  // integer count: order-independent
}

__global__ void k_vol_absmax(const float *z, const float *P, int64_t plane, int64_t pitch,
                             int D, int H, int W, float c1, float c2, float gamma,
                             unsigned *out_bits) {
    const int64_t n = (int64_t)D * H * W;
    const bool use_p = P != nullptr && gamma != 0.0f;
    float m = 0.0f;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = x / ((int64_t)H * W), r = x - k * H * W;
        const int i = (int)(r / W), j = (int)(r - (int64_t)i * W);
        const int64_t o = k * plane + (int64_t)i * pitch + j;
        const float aa = __fsub_rn(z[o], c1), bb = __fsub_rn(z[o], c2);
        float f = __fsub_rn(__fmul_rn(aa, aa), __fmul_rn(bb, bb));
        if (use_p) f = __fadd_rn(f, __fmul_rn(gamma, P[o]));
        m = fmaxf(m, fabsf(f));
    }
    for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out_bits, __float_as_uint(m));
}

// dense (D, H, W) <-> padded volume copies (one voxel per thread-iteration)
template <typename T>
__global__ void k_vol_copy(T *dst, const T *src, int64_t plane, int64_t pitch, int D, int H,
                           int W, int to_padded) {
    const int64_t n = (int64_t)D * H * W;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = x / ((int64_t)H * W), r = x - k * H * W;
        const int i = (int)(r / W), j = (int)(r - (int64_t)i * W);
        const int64_t o = k * plane + (int64_t)i * pitch + j;
        if (to_padded)
            dst[o] = src[x];
        else
            dst[x] = src[o];
    }
}

int64_t vol_tiles(int64_t H, int64_t W) {
    return ((W + VO_X - 1) / VO_X) * ((H + VO_Y - 1) / VO_Y);
}

cudaError_t launch_vol_step(const VolArgs &a, bool write_u, cudaStream_t s) {
    dim3 grid((a.W + VO_X - 1) / VO_X, (a.H + VO_Y - 1) / VO_Y, (a.D + a.kz - 1) / a.kz);
    // RDS_VOL_RPT=1 selects the one-row-per-thread kernel (A/B)
    static const bool one = getenv("RDS_VOL_RPT") && atoi(getenv("RDS_VOL_RPT")) == 1;
    if (one) {
        dim3 block(VT_X, VT_Y);
        if (write_u)
            k_vol_step<true><<<grid, block, 0, s>>>(a);
        else
            k_vol_step<false><<<grid, block, 0, s>>>(a);
    } else {
        dim3 block(VT_X, VT2_Y);
        if (write_u)
#ifdef RDS_VOL_2BAR
            k_vol_step2b<true><<<grid, block, 0, s>>>(a);
        else
            k_vol_step2b<false><<<grid, block, 0, s>>>(a);
#else
            k_vol_step2<true><<<grid, block, 0, s>>>(a);
        else
            k_vol_step2<false><<<grid, block, 0, s>>>(a);
#endif
    }
    return cudaGetLastError();
}

cudaError_t launch_vol_setup(const VolSetupArgs &a, cudaStream_t s) {
    k_vol_setup<<<148 * 8, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_vol_absmax(const float *z, const float *P, int64_t plane, int64_t pitch,
                              int D, int H, int W, float c1, float c2, float gamma,
                              unsigned *out_bits, cudaStream_t s) {
    k_vol_absmax<<<148 * 4, 256, 0, s>>>(z, P, plane, pitch, D, H, W, c1, c2, gamma, out_bits);
    return cudaGetLastError();
}

cudaError_t launch_vol_copy_f32(float *dst, const float *src, int64_t plane, int64_t pitch,
                                int D, int H, int W, int to_padded, cudaStream_t s) {
    k_vol_copy<float><<<148 * 8, 256, 0, s>>>(dst, src, plane, pitch, D, H, W, to_padded);
    return cudaGetLastError();
}

cudaError_t launch_vol_copy_u8(uint8_t *dst, const uint8_t *src, int64_t plane, int64_t pitch,
                               int D, int H, int W, int to_padded, cudaStream_t s) {
    k_vol_copy<uint8_t><<<148 * 8, 256, 0, s>>>(dst, src, plane, pitch, D, H, W, to_padded);
    return cudaGetLastError();
}

}  // namespace rds
