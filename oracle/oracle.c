/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the restricted-domain dual
 * iteration of arXiv 1807.11534 ("A Restricted-Domain Dual Formulation for Two-Phase Image
 * Segmentation").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no source, header, table or helper
 * with the CUDA product path (paper_1807_11534_b200/csrc/), and neither side includes the
 * other.
 *
 * Precision: the iteration runs in float64 (the paper fixes no precision).  The fitting term
 * (A1) and the band test (A2) are evaluated in float32 with a fixed operation order and no
 * contraction (build with -ffp-contract=off), because they decide integer labels and both
 * sides must take that decision in the same precision (reading R-A1).
 *
 * Citations are PAPER.md line numbers (section / equation) unless marked SPEC.md.
 * Readings of ambiguous passages are numbered as in DESIGN.md §3 (R-...).
 *
 * Parity pins: every function below is pinned by a -m "not gpu" test in tests/test_oracle_*.py
 * (closed forms, textbook identities, brute force, invariants).  The intermediate iterate
 * values themselves have no printed value in the paper: they are pinned only through those
 * closed forms, special cases and invariants.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define LAB_BG 0
#define LAB_FG 1
#define LAB_RD 2

#define IDX(i, j) ((int64_t)(i) * W + (j))

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Wall time of the last K-loop (solve_core's outer iterations only, not the labels, the     */
/* initialisation or the copies out) -- bench.py's CPU baseline times the loop alone         */
/* (BASELINE.md §3).  Measurement plumbing only; no part of the method.                       */
static double g_last_loop_s = 0.0;
double orc_last_loop_seconds(void) { return g_last_loop_s; }

static double wall_now(void) {
#ifdef _OPENMP
    return omp_get_wtime();
#else
    return 0.0;
#endif
}

/* ---------------------------------------------------------------------------------------- */
/* A1. Fitting term.  PAPER.md:31-33 (Eq. 2)  f = (z-c1)^2 - (z-c2)^2;                      */
/*     PAPER.md:35-37 (Eq. 3)  f = (z-c1)^2 - (z-c2)^2 + gamma P.                           */
/*     float32, order a=z-c1; b=z-c2; f=a*a-b*b; if gamma != 0: t=gamma*P; f=f+t.          */
/* ---------------------------------------------------------------------------------------- */
void orc_fitting(const float *z, const float *P, int64_t n, float c1, float c2, float gamma,
                 float *f) {
    for (int64_t k = 0; k < n; ++k) {
        float a = z[k] - c1;
        float b = z[k] - c2;
        float aa = a * a;
        float bb = b * b;
        float fk = aa - bb;
        if (gamma != 0.0f) {
            float t = gamma * P[k];
            fk = fk + t;
        }
        f[k] = fk;
    }
}

/* exact float32 max |f| (used to form the band threshold delta = delta_rel * max|f|). */
float orc_absmax(const float *f, int64_t n) {
    float m = 0.0f;
    for (int64_t k = 0; k < n; ++k) {
        float a = fabsf(f[k]);
        if (a > m) m = a;
    }
    return m;
}

/* ---------------------------------------------------------------------------------------- */
/* A2. Partition.  PAPER.md:74-83 (§3 set display):                                         */
/*   Fg = {f <= -q^},  Bg = {f >= q^},  RD = Omega \ Fg \ Bg.                               */
/*   Reading R-C7: RD <=> |f| < delta (strict); a pixel with |f| = delta is pinned; at       */
/*   delta = 0 the overlap f = 0 goes to Fg (consistent with H(0)=1, reading R-C2).          */
/* ---------------------------------------------------------------------------------------- */
void orc_labels(const float *f, int64_t n, float delta, uint8_t *lab) {
    for (int64_t k = 0; k < n; ++k) {
        if (fabsf(f[k]) < delta)
            lab[k] = LAB_RD;
        else if (f[k] <= 0.0f)
            lab[k] = LAB_FG;
        else
            lab[k] = LAB_BG;
    }
}

/* Active tiles: tile t = ti * ceil(W/tw) + tj is active iff it contains an RD pixel.        */
/* Writes the ascending list (if list != NULL) and returns the count.                       */
int64_t orc_tiles(const uint8_t *lab, int64_t H, int64_t W, int th, int tw, int32_t *list) {
    int64_t nti = (H + th - 1) / th, ntj = (W + tw - 1) / tw, cnt = 0;
    for (int64_t ti = 0; ti < nti; ++ti)
        for (int64_t tj = 0; tj < ntj; ++tj) {
            int active = 0;
            for (int64_t i = ti * th; i < (ti + 1) * th && i < H && !active; ++i)
                for (int64_t j = tj * tw; j < (tj + 1) * tw && j < W; ++j)
                    if (lab[IDX(i, j)] == LAB_RD) { active = 1; break; }
            if (active) {
                if (list) list[cnt] = (int32_t)(ti * ntj + tj);
                ++cnt;
            }
        }
    return cnt;
}

/* q -> q^ ("q^ is initially 0 and is increased until the selected value of */
/* q is satisfied").  Returns the smallest float32 q^ with #{|f| < q^} >= k, k = ceil(q n)     */
/* (double): q^ = nextafter(a_(k), +inf) with a_(k) the k-th smallest |f| (so pixels tied at   */
/* a_(k) join RD); q^ = 0 for k = 0.  Plain sort.                                 */
static int cmp_float(const void *a, const void *b) {
    float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

float orc_band_for_fraction(const float *f, int64_t n, double q) {
    int64_t k = (int64_t)ceil(q * (double)n);
    if (k > n) k = n;
    if (k <= 0) return 0.0f;
    float *a = (float *)malloc(sizeof(float) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) a[i] = fabsf(f[i]);
    qsort(a, (size_t)n, sizeof(float), cmp_float);
    float r = nextafterf(a[k - 1], INFINITY);
    free(a);
    return r;
}

/* ---------------------------------------------------------------------------------------- */
/* Discrete operators.  PAPER.md:70 defers them to Chambolle (2004) (not in the container);  */
/* reading R-C6 = SPEC.md:42, 51: forward-difference gradient with zero last row / column,   */
/* divergence = negative adjoint of the gradient.                                            */
/* ---------------------------------------------------------------------------------------- */
void orc_grad(const double *u, int64_t H, int64_t W, double *g1, double *g2) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < H; ++i)
        for (int64_t j = 0; j < W; ++j) {
            g1[IDX(i, j)] = (i < H - 1) ? u[IDX(i + 1, j)] - u[IDX(i, j)] : 0.0;
            g2[IDX(i, j)] = (j < W - 1) ? u[IDX(i, j + 1)] - u[IDX(i, j)] : 0.0;
        }
}

static inline double div_at(const double *p1, const double *p2, int64_t H, int64_t W,
                            int64_t i, int64_t j) {
    double d = (i < H - 1) ? p1[IDX(i, j)] : 0.0;
    d = d - ((i > 0) ? p1[IDX(i - 1, j)] : 0.0);
    d = d + ((j < W - 1) ? p2[IDX(i, j)] : 0.0);
    d = d - ((j > 0) ? p2[IDX(i, j - 1)] : 0.0);
    return d;
}

void orc_div(const double *p1, const double *p2, int64_t H, int64_t W, double *d) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < H; ++i)
        for (int64_t j = 0; j < W; ++j) d[IDX(i, j)] = div_at(p1, p2, H, W, i, j);
}

/* ---------------------------------------------------------------------------------------- */
/* Energies (double).                                                                        */
/*  E(w)  = TV(w) + lambda sum f w            PAPER.md:47-49 (Eq. 4), TV = sum |grad w|.     */
/*  D(p)  = sum min(0, lambda f + div p)      Lagrangian dual of Eq. 4 over u in [0,1]:       */
/*          TV(u) = max_{|p|<=1} <u, div p>, so E(u) >= <u, lambda f + div p> >= D(p).       */
/*  Sums are accumulated per row, then rows in order (deterministic for any thread count).   */
/* ---------------------------------------------------------------------------------------- */
static double tv_of(const double *w, int64_t H, int64_t W, double *rowbuf) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < H; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < W; ++j) {
            double a = (i < H - 1) ? w[IDX(i + 1, j)] - w[IDX(i, j)] : 0.0;
            double b = (j < W - 1) ? w[IDX(i, j + 1)] - w[IDX(i, j)] : 0.0;
            s += sqrt(a * a + b * b);
        }
        rowbuf[i] = s;
    }
    double t = 0.0;
    for (int64_t i = 0; i < H; ++i) t += rowbuf[i];
    return t;
}

double orc_tv(const double *w, int64_t H, int64_t W) {
    double *rb = (double *)malloc(sizeof(double) * (size_t)H);
    double t = tv_of(w, H, W, rb);
    free(rb);
    return t;
}

/* out[0]=E(v) out[1]=E(clamp(u,0,1)) out[2]=D(p) out[3]=E(v)-D(p) out[4]=TV(v)            */
/* out[5]=lambda*sum f v                                                                      */
void orc_energy(const float *f32, int64_t H, int64_t W, double lambda, const double *u,
                const double *v, const double *p1, const double *p2, double *out) {
    int64_t n = H * W;
    double *rb = (double *)malloc(sizeof(double) * (size_t)H);
    double *uc = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t k = 0; k < n; ++k) uc[k] = u[k] < 0.0 ? 0.0 : (u[k] > 1.0 ? 1.0 : u[k]);
    double tv_v = tv_of(v, H, W, rb);
    double tv_u = tv_of(uc, H, W, rb);
    double fit_v = 0.0, fit_u = 0.0, dual = 0.0;
    double *r2 = (double *)malloc(sizeof(double) * (size_t)H * 3);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < H; ++i) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int64_t j = 0; j < W; ++j) {
            double fk = (double)f32[IDX(i, j)];
            a += fk * v[IDX(i, j)];
            b += fk * uc[IDX(i, j)];
            double t = lambda * fk + div_at(p1, p2, H, W, i, j);
            c += (t < 0.0 ? t : 0.0);
        }
        r2[3 * i] = a;
        r2[3 * i + 1] = b;
        r2[3 * i + 2] = c;
    }
    for (int64_t i = 0; i < H; ++i) {
        fit_v += r2[3 * i];
        fit_u += r2[3 * i + 1];
        dual += r2[3 * i + 2];
    }
    out[0] = tv_v + lambda * fit_v;
    out[1] = tv_u + lambda * fit_u;
    out[2] = dual;
    out[3] = out[0] - out[2];
    out[4] = tv_v;
    out[5] = lambda * fit_v;
    free(rb);
    free(uc);
    free(r2);
}

/* ---------------------------------------------------------------------------------------- */
/* A3. The restricted-domain dual iteration.                                                 */
/*  Initialisation: u0 = H(-f) (reading R-C1 for the "-H(f)" typo at 113),      */
/*    H(0) = 1 (R-C2); v0 = u0 (R-C9); rho0 = 0.                              */
/*  One outer iteration, alternation rho -> u -> v:                    */
/*   rho-step, on RD (fixed point of Eq. 8, §3 form, reading R-C5):        */
/*      w   = div rho - v/theta          (full grid; rho = 0 off RD, Eq. 8 / reading R-C4)   */
/*      g   = grad w                                                                          */
/*      rho = (rho + tau g) / (1 + tau |g|)         on RD;   rho = 0 on Fg u Bg              */
/*   u-step (Eq. 7): u = v - theta div rho on RD; 1 on Fg; 0 on Bg.        */
/*   v-step (Eq. 9; r = f, reading R-C3):                                   */
/*      v = min(max(u - theta lambda f, 0), 1) on RD; 1 on Fg; 0 on Bg.                      */
/*  inner_steps (>=1) repeats the rho-step with v fixed (R-C9: default 1).                   */
/*  Optional warm start (v_init, p*_init, may be NULL): used on RD pixels only; pinned        */
/*  pixels take u0 / 0; p1 on the last row and p2 on the last column are zeroed (they are     */
/*  identically 0 under the iteration, reading R-C6).                                         */
/*  trace (may be NULL): per outer iteration `it` (0-based) writes ORC_NTRACE doubles:        */
/*    [0] max |rho|, [1] min v, [2] max v, [3] F^RD(u', v) (reading R-C12),                  */
/*    [4] E(v) - D(rho) (weak-duality gap).                                                   */
/* ---------------------------------------------------------------------------------------- */
#define ORC_NTRACE 5
int orc_ntrace(void) { return ORC_NTRACE; }

/* The iteration; with check_every > 0 also the stopping rule of PAPER.md:234-238 (§4),     */
/* "iterate until max{||u^l - u^(l-1)||, ||v^l - v^(l-1)||} <= delta is met at the l-th       */
/* iteration", evaluated after iterations check_every, 2 check_every, ... and at iters, with */
/* the Euclidean norm over the H*W pixels of unit area (norm = 0) or the RMS (norm = 1)      */
/* (reading R-F2).                                                                  */
static int solve_core(const float *f32, int64_t H, int64_t W, float delta, double lambda,
                      double theta, double tau, int iters, int inner_steps, const double *v_init,
                      const double *p1_init, const double *p2_init, double *u, double *v,
                      double *p1, double *p2, uint8_t *lab_out, double *trace, int check_every,
                      double tol, int norm, int *iters_done, double *residual) {
    if (H < 1 || W < 1 || iters < 0 || inner_steps < 1) return -1;
    int64_t n = H * W;
    uint8_t *lab = (uint8_t *)malloc((size_t)n);
    double *u0 = (double *)malloc(sizeof(double) * (size_t)n);
    double *f = (double *)malloc(sizeof(double) * (size_t)n);
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    double *vprev = (double *)malloc(sizeof(double) * (size_t)n);
    double *rb = (double *)malloc(sizeof(double) * (size_t)H * 2);
    double *uprev = check_every > 0 ? (double *)malloc(sizeof(double) * (size_t)n) : NULL;

    orc_labels(f32, n, delta, lab);
    for (int64_t k = 0; k < n; ++k) {
        f[k] = (double)f32[k];
        u0[k] = (f32[k] <= 0.0f) ? 1.0 : 0.0; /* H(-f), H(0)=1 */
    }
    for (int64_t i = 0; i < H; ++i)
        for (int64_t j = 0; j < W; ++j) {
            int64_t k = IDX(i, j);
            int rd = lab[k] == LAB_RD;
            v[k] = (rd && v_init) ? v_init[k] : u0[k];
            p1[k] = (rd && p1_init && i < H - 1) ? p1_init[k] : 0.0;
            p2[k] = (rd && p2_init && j < W - 1) ? p2_init[k] : 0.0;
            u[k] = u0[k];
        }

    /* touch the scratch planes before the timed loop (first-touch page faults are setup) */
    memset(w, 0, sizeof(double) * (size_t)n);
    memset(vprev, 0, sizeof(double) * (size_t)n);
    if (uprev) memset(uprev, 0, sizeof(double) * (size_t)n);
    if (iters_done) *iters_done = 0;
    if (residual) *residual = -1.0;
    const double t_loop0 = wall_now();
    for (int it = 0; it < iters; ++it) {
        /* v^(l-1) / u^(l-1) are needed only by the trace (F^RD) and the stopping rule */
        if (trace || check_every > 0) memcpy(vprev, v, sizeof(double) * (size_t)n);
        if (uprev) memcpy(uprev, u, sizeof(double) * (size_t)n);
        for (int s = 0; s < inner_steps; ++s) {
            /* w = div rho - v/theta on the full grid */
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j)
                    w[IDX(i, j)] = div_at(p1, p2, H, W, i, j) - v[IDX(i, j)] / theta;
            /* rho-step on RD (reads w only, so in-place update of rho is Jacobi) */
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j) {
                    int64_t k = IDX(i, j);
                    if (lab[k] != LAB_RD) {
                        p1[k] = 0.0;
                        p2[k] = 0.0;
                        continue;
                    }
                    double g1 = (i < H - 1) ? w[IDX(i + 1, j)] - w[k] : 0.0;
                    double g2 = (j < W - 1) ? w[IDX(i, j + 1)] - w[k] : 0.0;
                    double ng = sqrt(g1 * g1 + g2 * g2);
                    double den = 1.0 + tau * ng;
                    p1[k] = (p1[k] + tau * g1) / den;
                    p2[k] = (p2[k] + tau * g2) / den;
                }
        }
        /* u-step (Eq. 7) and v-step (Eq. 9) */
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                int64_t k = IDX(i, j);
                if (lab[k] != LAB_RD) {
                    u[k] = u0[k];
                    v[k] = u0[k];
                    continue;
                }
                double uk = v[k] - theta * div_at(p1, p2, H, W, i, j);
                u[k] = uk;
                double t = uk - theta * lambda * f[k];
                v[k] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
            }
        if (trace) {
            double *tr = trace + (int64_t)it * ORC_NTRACE;
            double pm = 0.0, vmin = INFINITY, vmax = -INFINITY;
            for (int64_t k = 0; k < n; ++k) {
                double a = sqrt(p1[k] * p1[k] + p2[k] * p2[k]);
                if (a > pm) pm = a;
                if (v[k] < vmin) vmin = v[k];
                if (v[k] > vmax) vmax = v[k];
            }
            tr[0] = pm;
            tr[1] = vmin;
            tr[2] = vmax;
            /* F^RD(u', v) = sum_{RD} |grad u'| + |u' - v|^2 / (2 theta) + lambda <f, v>,      */
            /* u' = v_prev - theta div rho on the full grid (reading R-C12).                  */
            double *up = w; /* reuse as scratch */
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j)
                    up[IDX(i, j)] = vprev[IDX(i, j)] - theta * div_at(p1, p2, H, W, i, j);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < H; ++i) {
                double a = 0.0, b = 0.0;
                for (int64_t j = 0; j < W; ++j) {
                    int64_t k = IDX(i, j);
                    if (lab[k] == LAB_RD) {
                        double g1 = (i < H - 1) ? up[IDX(i + 1, j)] - up[k] : 0.0;
                        double g2 = (j < W - 1) ? up[IDX(i, j + 1)] - up[k] : 0.0;
                        a += sqrt(g1 * g1 + g2 * g2);
                    }
                    double d = up[k] - v[k];
                    b += d * d / (2.0 * theta) + lambda * f[k] * v[k];
                }
                rb[2 * i] = a;
                rb[2 * i + 1] = b;
            }
            double F = 0.0;
            for (int64_t i = 0; i < H; ++i) F += rb[2 * i] + rb[2 * i + 1];
            tr[3] = F;
            double e[6];
            orc_energy(f32, H, W, lambda, u, v, p1, p2, e);
            tr[4] = e[3];
        }
        if (iters_done) *iters_done = it + 1;
        if (check_every > 0 && ((it + 1) % check_every == 0 || it + 1 == iters)) {
            /* row sums in a fixed order: the result does not depend on the thread count */
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < H; ++i) {
                double a = 0.0, b = 0.0;
                for (int64_t j = 0; j < W; ++j) {
                    int64_t k = IDX(i, j);
                    double du = u[k] - uprev[k], dv = v[k] - vprev[k];
                    a += du * du;
                    b += dv * dv;
                }
                rb[2 * i] = a;
                rb[2 * i + 1] = b;
            }
            double su = 0.0, sv = 0.0;
            for (int64_t i = 0; i < H; ++i) {
                su += rb[2 * i];
                sv += rb[2 * i + 1];
            }
            double nd = norm ? (double)n : 1.0;
            double ru = sqrt(su / nd), rv = sqrt(sv / nd);
            double r = ru > rv ? ru : rv;
            if (residual) *residual = r;
            if (r <= tol) break;
        }
    }
    g_last_loop_s = wall_now() - t_loop0;
    if (lab_out) memcpy(lab_out, lab, (size_t)n);
    free(lab);
    free(u0);
    free(f);
    free(w);
    free(vprev);
    free(rb);
    free(uprev);
    return 0;
}

int orc_solve(const float *f32, int64_t H, int64_t W, float delta, double lambda,
              double theta, double tau, int iters, int inner_steps, const double *v_init,
              const double *p1_init, const double *p2_init, double *u, double *v, double *p1,
              double *p2, uint8_t *lab_out, double *trace) {
    return solve_core(f32, H, W, delta, lambda, theta, tau, iters, inner_steps, v_init,
                      p1_init, p2_init, u, v, p1, p2, lab_out, trace, 0, 0.0, 0, NULL, NULL);
}

/* orc_solve with the stopping rule: stops at the first check with residual <= tol, else at  */
/* max_iters.  Writes the iterations done and the residual of the last check.                */
int orc_solve_tol(const float *f32, int64_t H, int64_t W, float delta, double lambda,
                  double theta, double tau, int max_iters, int check_every, double tol,
                  int norm, double *u, double *v, double *p1, double *p2, uint8_t *lab_out,
                  int *iters_done, double *residual) {
    if (check_every < 1 || max_iters < 1 || !(tol >= 0.0)) return -1;
    return solve_core(f32, H, W, delta, lambda, theta, tau, max_iters, 1, NULL, NULL, NULL, u,
                      v, p1, p2, lab_out, NULL, check_every, tol, norm, iters_done, residual);
}

/* ---------------------------------------------------------------------------------------- */
/* The plain, unrestricted Bresson/Chambolle iteration of PAPER.md:58-70 (§2.1), written    */
/* separately with no partition logic.  Pin: orc_solve with delta = +inf must reproduce it   */
/* bit for bit ("For q=1 ... we consider the problem in a conventional manner";  */
/* SPEC.md:302).                                                                              */
/* ---------------------------------------------------------------------------------------- */
int orc_solve_plain(const float *f32, int64_t H, int64_t W, double lambda, double theta,
                    double tau, int iters, double *u, double *v, double *p1, double *p2) {
    if (H < 1 || W < 1 || iters < 0) return -1;
    int64_t n = H * W;
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t k = 0; k < n; ++k) {
        v[k] = (f32[k] <= 0.0f) ? 1.0 : 0.0;
        u[k] = v[k];
        p1[k] = 0.0;
        p2[k] = 0.0;
    }
    for (int it = 0; it < iters; ++it) {
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                double d = 0.0;
                if (i < H - 1) d += p1[IDX(i, j)];
                if (i > 0) d -= p1[IDX(i - 1, j)];
                if (j < W - 1) d += p2[IDX(i, j)];
                if (j > 0) d -= p2[IDX(i, j - 1)];
                w[IDX(i, j)] = d - v[IDX(i, j)] / theta;
            }
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                double g1 = 0.0, g2 = 0.0;
                if (i < H - 1) g1 = w[IDX(i + 1, j)] - w[IDX(i, j)];
                if (j < W - 1) g2 = w[IDX(i, j + 1)] - w[IDX(i, j)];
                double den = 1.0 + tau * sqrt(g1 * g1 + g2 * g2);
                p1[IDX(i, j)] = (p1[IDX(i, j)] + tau * g1) / den;
                p2[IDX(i, j)] = (p2[IDX(i, j)] + tau * g2) / den;
            }
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                double d = 0.0;
                if (i < H - 1) d += p1[IDX(i, j)];
                if (i > 0) d -= p1[IDX(i - 1, j)];
                if (j < W - 1) d += p2[IDX(i, j)];
                if (j > 0) d -= p2[IDX(i, j - 1)];
                double uk = v[IDX(i, j)] - theta * d;
                u[IDX(i, j)] = uk;
                double t = uk - theta * lambda * (double)f32[IDX(i, j)];
                v[IDX(i, j)] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
            }
    }
    free(w);
    return 0;
}

/* ---------------------------------------------------------------------------------------- */
/* Chambolle inner problem with v fixed (restricted support).  Runs `steps` rho-steps of     */
/* PAPER.md:138-141 on RD and records obj[s] = || div rho - v/theta ||^2 after each step.    */
/* Pin: non-increasing for tau <= 1/8 (Chambolle 2004's fixed-point descent; the restricted   */
/* support is a coordinate subset, reading R-C12).                                            */
/* ---------------------------------------------------------------------------------------- */
int orc_inner(const float *f32, int64_t H, int64_t W, float delta, double theta, double tau,
              int steps, const double *v, double *p1, double *p2, double *obj) {
    int64_t n = H * W;
    uint8_t *lab = (uint8_t *)malloc((size_t)n);
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    orc_labels(f32, n, delta, lab);
    for (int64_t i = 0; i < H; ++i)
        for (int64_t j = 0; j < W; ++j) {
            int64_t k = IDX(i, j);
            if (lab[k] != LAB_RD || i == H - 1) p1[k] = 0.0;
            if (lab[k] != LAB_RD || j == W - 1) p2[k] = 0.0;
        }
    for (int s = 0; s < steps; ++s) {
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j)
                w[IDX(i, j)] = div_at(p1, p2, H, W, i, j) - v[IDX(i, j)] / theta;
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                int64_t k = IDX(i, j);
                if (lab[k] != LAB_RD) continue;
                double g1 = (i < H - 1) ? w[IDX(i + 1, j)] - w[k] : 0.0;
                double g2 = (j < W - 1) ? w[IDX(i, j + 1)] - w[k] : 0.0;
                double den = 1.0 + tau * sqrt(g1 * g1 + g2 * g2);
                p1[k] = (p1[k] + tau * g1) / den;
                p2[k] = (p2[k] + tau * g2) / den;
            }
        double o = 0.0;
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                double d = div_at(p1, p2, H, W, i, j) - v[IDX(i, j)] / theta;
                o += d * d;
            }
        obj[s] = o;
    }
    free(lab);
    free(w);
    return 0;
}

/* ---------------------------------------------------------------------------------------- */
/* f4: the same method on 3-D volumes (§5: "extension to 3D").  A volume is    */
/* D planes x H rows x W columns, plane-major.  The discrete operators extend reading R-C6   */
/* axis by axis (reading R-F4): forward differences with a zero last plane / row / column,  */
/* div = -grad^T, components rho1 (rows, i), rho2 (columns, j), rho3 (planes, k).           */
/* Labels and the fitting term are per voxel (orc_fitting / orc_labels with n = D H W).     */
/* ---------------------------------------------------------------------------------------- */
#define IDX3(k, i, j) (((int64_t)(k) * H + (i)) * W + (j))

void orc_grad3(const double *u, int64_t D, int64_t H, int64_t W, double *g1, double *g2,
               double *g3) {
    for (int64_t k = 0; k < D; ++k)
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) {
                int64_t x = IDX3(k, i, j);
                g1[x] = (i < H - 1) ? u[IDX3(k, i + 1, j)] - u[x] : 0.0;
                g2[x] = (j < W - 1) ? u[IDX3(k, i, j + 1)] - u[x] : 0.0;
                g3[x] = (k < D - 1) ? u[IDX3(k + 1, i, j)] - u[x] : 0.0;
            }
}

static inline double div3_at(const double *p1, const double *p2, const double *p3, int64_t D,
                             int64_t H, int64_t W, int64_t k, int64_t i, int64_t j) {
    double d = (i < H - 1) ? p1[IDX3(k, i, j)] : 0.0;
    d = d - ((i > 0) ? p1[IDX3(k, i - 1, j)] : 0.0);
    d = d + ((j < W - 1) ? p2[IDX3(k, i, j)] : 0.0);
    d = d - ((j > 0) ? p2[IDX3(k, i, j - 1)] : 0.0);
    d = d + ((k < D - 1) ? p3[IDX3(k, i, j)] : 0.0);
    d = d - ((k > 0) ? p3[IDX3(k - 1, i, j)] : 0.0);
    return d;
}

void orc_div3(const double *p1, const double *p2, const double *p3, int64_t D, int64_t H,
              int64_t W, double *d) {
    for (int64_t k = 0; k < D; ++k)
        for (int64_t i = 0; i < H; ++i)
            for (int64_t j = 0; j < W; ++j) d[IDX3(k, i, j)] = div3_at(p1, p2, p3, D, H, W, k, i, j);
}

/* The restricted-domain iteration of orc_solve (§2.1 + §3, Eq. 7-9) on a volume. */
int orc_solve3(const float *f32, int64_t D, int64_t H, int64_t W, float delta, double lambda,
               double theta, double tau, int iters, double *u, double *v, double *p1,
               double *p2, double *p3, uint8_t *lab_out) {
    if (D < 1 || H < 1 || W < 1 || iters < 0) return -1;
    int64_t n = D * H * W;
    uint8_t *lab = (uint8_t *)malloc((size_t)n);
    double *u0 = (double *)malloc(sizeof(double) * (size_t)n);
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    orc_labels(f32, n, delta, lab);
    for (int64_t x = 0; x < n; ++x) {
        u0[x] = (f32[x] <= 0.0f) ? 1.0 : 0.0; /* H(-f), H(0) = 1 */
        u[x] = v[x] = u0[x];
        p1[x] = p2[x] = p3[x] = 0.0;
    }
    for (int it = 0; it < iters; ++it) {
        /* w = div rho - v/theta on the full grid */
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < D; ++k)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j)
                    w[IDX3(k, i, j)] =
                        div3_at(p1, p2, p3, D, H, W, k, i, j) - v[IDX3(k, i, j)] / theta;
        /* rho-step on RD, 0 on Fg u Bg (Eq. 8) */
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < D; ++k)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j) {
                    int64_t x = IDX3(k, i, j);
                    if (lab[x] != LAB_RD) {
                        p1[x] = p2[x] = p3[x] = 0.0;
                        continue;
                    }
                    double g1 = (i < H - 1) ? w[IDX3(k, i + 1, j)] - w[x] : 0.0;
                    double g2 = (j < W - 1) ? w[IDX3(k, i, j + 1)] - w[x] : 0.0;
                    double g3 = (k < D - 1) ? w[IDX3(k + 1, i, j)] - w[x] : 0.0;
                    double den = 1.0 + tau * sqrt(g1 * g1 + g2 * g2 + g3 * g3);
                    p1[x] = (p1[x] + tau * g1) / den;
                    p2[x] = (p2[x] + tau * g2) / den;
                    p3[x] = (p3[x] + tau * g3) / den;
                }
        /* u-step (Eq. 7), v-step (Eq. 9) */
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < D; ++k)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j) {
                    int64_t x = IDX3(k, i, j);
                    if (lab[x] != LAB_RD) {
                        u[x] = v[x] = u0[x];
                        continue;
                    }
                    double ux = v[x] - theta * div3_at(p1, p2, p3, D, H, W, k, i, j);
                    u[x] = ux;
                    double t = ux - theta * lambda * (double)f32[x];
                    v[x] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
                }
    }
    if (lab_out) memcpy(lab_out, lab, (size_t)n);
    free(lab);
    free(u0);
    free(w);
    return 0;
}

/* The unrestricted 3-D iteration written out separately (no partition logic), the twin    */
/* orc_solve3 must reproduce bit for bit at delta = +inf.                                    */
int orc_solve3_plain(const float *f32, int64_t D, int64_t H, int64_t W, double lambda,
                     double theta, double tau, int iters, double *u, double *v, double *p1,
                     double *p2, double *p3) {
    if (D < 1 || H < 1 || W < 1 || iters < 0) return -1;
    int64_t n = D * H * W;
    double *w = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t x = 0; x < n; ++x) {
        v[x] = (f32[x] <= 0.0f) ? 1.0 : 0.0;
        u[x] = v[x];
        p1[x] = p2[x] = p3[x] = 0.0;
    }
    for (int it = 0; it < iters; ++it) {
        for (int64_t k = 0; k < D; ++k)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j) {
                    double d = 0.0;
                    if (i < H - 1) d += p1[IDX3(k, i, j)];
                    if (i > 0) d -= p1[IDX3(k, i - 1, j)];
                    if (j < W - 1) d += p2[IDX3(k, i, j)];
                    if (j > 0) d -= p2[IDX3(k, i, j - 1)];
                    if (k < D - 1) d += p3[IDX3(k, i, j)];
                    if (k > 0) d -= p3[IDX3(k - 1, i, j)];
                    w[IDX3(k, i, j)] = d - v[IDX3(k, i, j)] / theta;
                }
        for (int64_t k = 0; k < D; ++k)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j) {
                    int64_t x = IDX3(k, i, j);
                    double g1 = 0.0, g2 = 0.0, g3 = 0.0;
                    if (i < H - 1) g1 = w[IDX3(k, i + 1, j)] - w[x];
                    if (j < W - 1) g2 = w[IDX3(k, i, j + 1)] - w[x];
                    if (k < D - 1) g3 = w[IDX3(k + 1, i, j)] - w[x];
                    double den = 1.0 + tau * sqrt(g1 * g1 + g2 * g2 + g3 * g3);
                    p1[x] = (p1[x] + tau * g1) / den;
                    p2[x] = (p2[x] + tau * g2) / den;
                    p3[x] = (p3[x] + tau * g3) / den;
                }
        for (int64_t k = 0; k < D; ++k)
            for (int64_t i = 0; i < H; ++i)
                for (int64_t j = 0; j < W; ++j) {
                    int64_t x = IDX3(k, i, j);
                    double d = 0.0;
                    if (i < H - 1) d += p1[x];
                    if (i > 0) d -= p1[IDX3(k, i - 1, j)];
                    if (j < W - 1) d += p2[x];
                    if (j > 0) d -= p2[IDX3(k, i, j - 1)];
                    if (k < D - 1) d += p3[x];
                    if (k > 0) d -= p3[IDX3(k - 1, i, j)];
                    double ux = v[x] - theta * d;
                    u[x] = ux;
                    double t = ux - theta * lambda * (double)f32[x];
                    v[x] = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
                }
    }
    free(w);
    return 0;
}
