// k_fp64.cu -- the float64 mode of librds (sm_100a): the same restricted-domain iteration in
// double precision, for the paper's ground-truth protocol (§4): "For
// delta = 10^-10 we set u^GT(x) = u^(l) in the original dual formulation", then E1 (Tanimoto
// of the thresholded results) and E2 (L2 difference) against a restricted solve.
//
// A tolerance of 1e-10 in the stopping rule is below float32 resolution, so this mode keeps
// every state array in float64 and uses correctly rounded sqrt / division with no FMA
// contraction (explicit _rn intrinsics), each formula evaluated left to right as written:
//   w   = div rho - v / theta
//   rho = (rho + tau grad w) / (1 + tau |grad w|) on RD, 0 on Fg u Bg   (Eq. 8)
//   u   = v - theta div rho on RD, u0 elsewhere                 (Eq. 7)
//   v   = min(max(u - (theta lambda) f, 0), 1) on RD, u0 elsewhere (Eq. 9)
// with div rho = ((rho1 - rho1(i-1,j)) + rho2) - rho2(i,j-1) (reading R-C6).  Throughput is
// not the first concern here (this is the reference-quality solver of the evaluation protocol,
// run on the paper's 128 x 128 images), so it works on natural-order double planes (padded
// like the float planes; the frame holds zeros), one persistent cooperative launch per solve.
#include <math.h>

#include "internal.h"

namespace rds {

__device__ __forceinline__ float fit32(float z, float P, float c1, float c2, float gamma,
                                       bool use_p) {
    const float a = __fsub_rn(z, c1), b = __fsub_rn(z, c2);
    float f = __fsub_rn(__fmul_rn(a, a), __fmul_rn(b, b));
    if (use_p) f = __fadd_rn(f, __fmul_rn(gamma, P));
    return f;
}

// div rho at (i, j) in the padded double planes (frame = 0; rho1 on row H-1 and rho2 on
// column W-1 are identically 0, so no bounds tests are needed)
__device__ __forceinline__ double div64(const double *p1, const double *p2, int64_t o,
                                        int64_t pitch) {
    double d = __dsub_rn(p1[o], p1[o - pitch]);
    d = __dadd_rn(d, p2[o]);
    return __dsub_rn(d, p2[o - 1]);
}

__global__ void k64_init(const F64Args a) {
    const int64_t n = (int64_t)a.H * a.W;
    const bool use_p = a.P != nullptr && a.gamma != 0.0f;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(k / a.W), j = (int)(k - (int64_t)i * a.W);
        const int64_t o = (int64_t)i * a.pitch + j;
        const float f = fit32(a.z[o], use_p ? a.P[o] : 0.0f, a.c1, a.c2, a.gamma, use_p);
        const bool rd = fabsf(f) < a.delta;             // RD <=> |f| < delta (R-C7)
        const double u0 = f <= 0.0f ? 1.0 : 0.0;        // H(-f), H(0) = 1
        a.f[o] = (double)f;
        a.lab[o] = rd ? 2 : (f <= 0.0f ? 1 : 0);
        a.u[o] = u0;
        a.v[o] = u0;
        if (a.v2) a.v2[o] = u0;  // the persistent solve's second v buffer
        a.p1[0][o] = a.p1[1][o] = 0.0;
        a.p2[0][o] = a.p2[1][o] = 0.0;
    }
}

// ---------------------------------------------------------------------------------------
// Persistent form (rds_solve_gt): ONE cooperative launch runs the whole solve, a grid barrier
// between iterations.  Pass k at pixel x (on RD; pinned pixels never change) computes, from
// rho^k and v^{k-1}, the u/v step of iteration k at x and at its two forward neighbours
// (recomputed so one barrier per iteration suffices), then w^k and rho^{k+1}(x) -- exactly
// operations written out at the top of this file, each in the order written, so the iterates
// are the same bits as the fp64 oracle's.  At a check iteration the CTAs publish fixed-order partial sums of
// (u^l - u^{l-1})^2, (v^l - v^{l-1})^2 and, after the barrier, all form the same total and take
// the same stop decision.
// ---------------------------------------------------------------------------------------

namespace {

__device__ __forceinline__ void gbar(unsigned long long *bar, unsigned long long k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned long long target = k * gridDim.x;
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ double wsum(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// fixed-order CTA sum of two doubles (valid in thread 0)
__device__ __forceinline__ void cta2(double &a, double &b, double (*sh)[F64P_THREADS / 32]) {
    a = wsum(a);
    b = wsum(b);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = a;
        sh[1][threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a = b = 0.0;
        for (int w = 0; w < F64P_THREADS / 32; ++w) {
            a += sh[0][w];
            b += sh[1][w];
        }
    }
}

// v^k at an RD pixel y from v^{k-1}(y) and div rho^k(y): u = v - theta div rho, then the clamp
__device__ __forceinline__ double v_step(double vp, double d, double f, double theta,
                                         double theta_lambda, double *u_out) {
    const double u = __dsub_rn(vp, __dmul_rn(theta, d));
    const double t = __dsub_rn(u, __dmul_rn(theta_lambda, f));
    *u_out = u;
    return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}

}  // namespace

// stop decision after a check (all CTAs, same total in the same order); returns fire
__device__ __forceinline__ bool f64_check(const F64Persist &q, double su, double sv, int k,
                                          unsigned long long &nbar, int &nchk,
                                          double (*sh)[F64P_THREADS / 32], int *stop_s) {
    // two buffers alternating by check parity: with checks one iteration apart no barrier
    // separates a fast CTA's write for check c+1 from a slow CTA's read for check c
    double *part = q.part + (nchk++ & 1) * 2 * F64P_MAX_GRID;
    cta2(su, sv, sh);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = su;
        part[2 * blockIdx.x + 1] = sv;
    }
    gbar(q.bar, ++nbar);
    double tu = 0.0, tv = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
        tu += __ldcg(part + 2 * b);
        tv += __ldcg(part + 2 * b + 1);
    }
    cta2(tu, tv, sh);
    if (threadIdx.x == 0) {
        const double r = fmax(sqrt(tu / q.norm_div), sqrt(tv / q.norm_div));
        const bool conv = r <= q.tol, fire = conv || k >= q.max_iters;
        *stop_s = fire;
        if (blockIdx.x == 0) {
            StopRecord *rec = q.a.stop;
            rec->it = k;
            rec->residual = r;
            rec->checks += 1;
            if (fire) {
                rec->iters = k;
                rec->converged = conv ? 1 : 0;
                rec->flag = 1;
            }
        }
    }
    __syncthreads();
    return *stop_s != 0;
}

__global__ void __launch_bounds__(F64P_THREADS) k64_persist(const F64Persist q) {
    const F64Args &a = q.a;
    const int64_t n = (int64_t)a.H * a.W, P = a.pitch;
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = blockIdx.x * chunk, k1 = min(n, k0 + chunk);
    const double theta = a.theta, tau = a.tau, tl = a.theta_lambda;
    __shared__ double sh[2][F64P_THREADS / 32];
    __shared__ int stop_s;
    const int K = q.max_iters, m = q.check_every;
    unsigned long long nbar = 0;
    int nchk = 0;
    for (int k = 0; k <= K; ++k) {
        const bool odd = k & 1;
        const double *p1 = odd ? a.p1[1] : a.p1[0], *p2 = odd ? a.p2[1] : a.p2[0];
        double *q1 = odd ? a.p1[0] : a.p1[1], *q2 = odd ? a.p2[0] : a.p2[1];
        // v^{k-1} in buffer (k-1)&1 (pass 0: v^0 in buffer 0); v^k goes to buffer k&1
        const double *vp = (k == 0 || odd) ? q.v[0] : q.v[1];
        double *vo = odd ? q.v[1] : q.v[0];
        const bool chk = k >= 1 && (k % m == 0 || k == K);
        double su = 0.0, sv = 0.0;
        for (int64_t x = k0 + threadIdx.x; x < k1; x += blockDim.x) {
            const int i = (int)(x / a.W), j = (int)(x - (int64_t)i * a.W);
            const int64_t o = (int64_t)i * P + j;
            if (a.lab[o] != 2) continue;  // pinned: rho = 0 and u = v = u0 for good
            const double dx = div64(p1, p2, o, P);
            double ux = 0.0, vx = vp[o];
            if (k >= 1) vx = v_step(vp[o], dx, a.f[o], theta, tl, &ux);
            if (k >= 1) {
                if (chk) {
                    const double du = __dsub_rn(ux, a.u[o]), dv = __dsub_rn(vx, vp[o]);
                    su = __fma_rn(du, du, su);
                    sv = __fma_rn(dv, dv, sv);
                }
                a.u[o] = ux;
                vo[o] = vx;
            }
            if (k == K) continue;
            // rho-step of iteration k+1: w = div rho - v / theta, g = grad w, the fixed point
            const double w = __dsub_rn(dx, __ddiv_rn(vx, theta));
            double g1 = 0.0, g2 = 0.0;
            if (i < a.H - 1) {
                const int64_t y = o + P;
                const double dy = div64(p1, p2, y, P);
                double vy = vp[y], uy;
                if (k >= 1 && a.lab[y] == 2) vy = v_step(vp[y], dy, a.f[y], theta, tl, &uy);
                g1 = __dsub_rn(__dsub_rn(dy, __ddiv_rn(vy, theta)), w);
            }
            if (j % a.img_w != a.img_w - 1) {
                const int64_t y = o + 1;
                const double dy = div64(p1, p2, y, P);
                double vy = vp[y], uy;
                if (k >= 1 && a.lab[y] == 2) vy = v_step(vp[y], dy, a.f[y], theta, tl, &uy);
                g2 = __dsub_rn(__dsub_rn(dy, __ddiv_rn(vy, theta)), w);
            }
            const double ng = __dsqrt_rn(__dadd_rn(__dmul_rn(g1, g1), __dmul_rn(g2, g2)));
            const double den = __dadd_rn(1.0, __dmul_rn(tau, ng));
            q1[o] = __ddiv_rn(__dadd_rn(p1[o], __dmul_rn(tau, g1)), den);
            q2[o] = __ddiv_rn(__dadd_rn(p2[o], __dmul_rn(tau, g2)), den);
        }
        if (chk) {
            if (f64_check(q, su, sv, k, nbar, nchk, sh, &stop_s)) break;
        } else if (k < K) {
            gbar(q.bar, ++nbar);
        }
    }
}

cudaError_t launch_f64_persist(const F64Persist &q, int n_sm, cudaStream_t s) {
    // up to 4 CTAs per SM (the occupancy limit at 64 registers): latency hiding for the
    // dependent fp64 division chains outweighs the extra barrier arrivals (measured: C1 u^GT
    // 27.8 us per iteration at 4 vs 42.8 at 2; a two-phase variant without the neighbour
    // recomputation was slower at both C0 and C1)
    static int per_sm = 0;
    if (per_sm <= 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k64_persist, F64P_THREADS,
                                                          0) != cudaSuccess ||
            per_sm < 1) {
            (void)cudaGetLastError();
            per_sm = 1;
        }
        if (per_sm > 4) per_sm = 4;
    }
    const int64_t n = (int64_t)q.a.H * q.a.W;
    int g = per_sm * n_sm;
    const int64_t need = (n + F64P_THREADS - 1) / F64P_THREADS;
    if (g > need) g = (int)need;
    if (g > F64P_MAX_GRID) g = F64P_MAX_GRID;
    cudaError_t e = cudaMemsetAsync(q.bar, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    void *args[] = {const_cast<F64Persist *>(&q)};
    return cudaLaunchCooperativeKernel((const void *)k64_persist, dim3(g), dim3(F64P_THREADS),
                                       args, 0, s);
}

int f64_grid(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return (int)(g < F64_BLOCKS ? g : F64_BLOCKS);
}
cudaError_t launch_f64_init(const F64Args &a, cudaStream_t s) {
    k64_init<<<f64_grid((int64_t)a.H * a.W), 256, 0, s>>>(a);
    return cudaGetLastError();
}

// E1 = N(GT n Omega) / N(GT u Omega) with GT = [u_gt > eps], Omega = [u > eps] (1 when both
// are empty, reading R-C15), E2 = sum (u - u_gt)^2 over pixels of unit area.
// Integer counts and fixed-order double sums: deterministic.
__global__ void __launch_bounds__(256) k_compare(const float *u, const double *ugt,
                                                 int64_t pitch, int H, int W, float eps,
                                                 double *part) {
    const int64_t n = (int64_t)H * W;
    long long in = 0, un = 0;
    double e2 = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(k / W), j = (int)(k - (int64_t)i * W);
        const int64_t o = (int64_t)i * pitch + j;
        const double a = (double)u[o], g = ugt[o];
        const bool om = u[o] > eps, gt = g > (double)eps;
        in += om && gt;
        un += om || gt;
        const double d = __dsub_rn(a, g);
        e2 = __fma_rn(d, d, e2);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        in += __shfl_xor_sync(0xffffffffu, in, off);
        un += __shfl_xor_sync(0xffffffffu, un, off);
        e2 += __shfl_xor_sync(0xffffffffu, e2, off);
    }
    __shared__ double sh[3][8];
    if ((threadIdx.x & 31) == 0) {
        sh[0][threadIdx.x >> 5] = (double)in;
        sh[1][threadIdx.x >> 5] = (double)un;
        sh[2][threadIdx.x >> 5] = e2;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sh[threadIdx.x][w];
        part[3 * blockIdx.x + threadIdx.x] = t;
    }
}

__global__ void k_compare_final(const double *part, int nb, double *out) {
    if (threadIdx.x == 0) {
        double in = 0.0, un = 0.0, e2 = 0.0;
        for (int b = 0; b < nb; ++b) {
            in += part[3 * b];
            un += part[3 * b + 1];
            e2 += part[3 * b + 2];
        }
        out[0] = un > 0.0 ? in / un : 1.0;
        out[1] = e2;
    }
}

cudaError_t launch_compare(const float *u, const double *ugt, int64_t pitch, int H, int W,
                           float eps, double *part, double *out, cudaStream_t s) {
    const int g = f64_grid((int64_t)H * W);
    k_compare<<<g, 256, 0, s>>>(u, ugt, pitch, H, W, eps, part);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_compare_final<<<1, 32, 0, s>>>(part, g, out);
    return cudaGetLastError();
}

}  // namespace rds
