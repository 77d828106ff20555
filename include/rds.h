/*
 * rds.h -- C ABI of librds: the restricted-domain dual iteration of arXiv 1807.11534
 * ("A Restricted-Domain Dual Formulation for Two-Phase Image Segmentation") on one B200
 * (sm_100a).  Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *
 * The method (PAPER.md line numbers, section / equation):
 *   fitting term   f = (z - c1)^2 - (z - c2)^2 + gamma P          PAPER.md:31-37 (Eq. 2, 3)
 *   partition      Fg = {f <= -delta}, Bg = {f >= delta}, RD = rest  PAPER.md:74-83 (§3)
 *                  (RD <=> |f| < delta; reading R-C7)
 *   init           u0 = v0 = H(-f) (H(0) = 1), rho0 = 0
 *   rho-step (RD)  rho <- (rho + tau grad w) / (1 + tau |grad w|),
 *                  w = div rho - v/theta; rho = 0 on Fg u Bg       PAPER.md:129-141 (Eq. 8)
 *   u-step         u = v - theta div rho on RD; 1 on Fg; 0 on Bg   PAPER.md:119-128 (Eq. 7)
 *   v-step         v = min(max(u - theta lambda f, 0), 1) on RD;
 *                  1 on Fg; 0 on Bg                                 PAPER.md:146-155 (Eq. 9)
 *   threshold      mask = [u > 0.5]
 *   Discrete grad = forward differences with zero last row/col, div = -grad^T
 *   (PAPER.md:70 defers to Chambolle 2004; reading R-C6).
 *
 * Layout conventions: every image argument is H x W, row-major (row i, column j), densely
 * packed (row stride W elements).  `on_device` = 1 means the pointer is CUDA device memory
 * (e.g. a torch CUDA tensor's data_ptr), 0 means host memory.  The library copies inputs into
 * its own storage; the caller keeps ownership of every pointer it passes and may reuse it as
 * soon as the call returns (host copies are synchronous; device copies are stream-ordered on
 * the handle's stream, so a device buffer must stay valid until that stream reaches the copy).
 *
 * Errors: every call returns an int, RDS_OK (0) or a negative code; no call throws across the
 * ABI.  rds_last_error() gives a message for the last failure on that handle.  A handle is not
 * thread-safe; distinct handles are independent.  Results are deterministic: identical inputs
 * produce bit-identical outputs (no atomics on any output path).
 */
#ifndef RDS_H_
#define RDS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RDS_OK 0
#define RDS_EINVAL (-1)  /* invalid argument (NULL, size, parameter range, non-finite data) */
#define RDS_ESTATE (-2)  /* call out of order (e.g. solve before image/fitting, get before solve) */
#define RDS_ECUDA (-3)   /* a CUDA runtime call or kernel launch failed */
#define RDS_ENOMEM (-4)  /* device allocation failed */

/* Pixel labels: 0 = Bg (pinned u = v = 0), 1 = Fg (pinned u = v = 1),
 * 2 = RD (iterated). */
#define RDS_LABEL_BG 0
#define RDS_LABEL_FG 1
#define RDS_LABEL_RD 2

/* Active-tile granularity exported by rds_get_active_tiles (see rds_tile_shape). */
#define RDS_TILE_H 32
#define RDS_TILE_W 32

typedef struct rds_handle rds_t;

/* Energies of the current state, all double (rds_energy).
 *  E_v   = TV(v) + lambda sum f v            (Eq. 4, at w = v)
 *  E_u   = TV(c(u)) + lambda sum f c(u),     c(u) = min(max(u,0),1)
 *  D_p   = sum min(0, lambda f + div rho)    (Lagrangian dual of Eq. 4 over u in [0,1])
 *  gap   = E_v - D_p  (>= 0 by weak duality whenever |rho| <= 1)
 *  TV_v, fit_v = lambda sum f v : the two parts of E_v.
 *  F_rd  = sum_{RD} |grad u'| + sum |u' - v|^2 / (2 theta) + lambda sum f v with
 *          u' = v_prev - theta div rho (the last u on RD, u0 - theta div rho off RD): the
 *          restricted functional that the iteration decreases (reading R-C12). */
typedef struct {
    double E_v, E_u, D_p, gap, TV_v, fit_v, F_rd;
} rds_energy_t;

/* Statistics of the last rds_solve. Times are CUDA-event times on the handle's stream and are
 * only filled when RDS_OPT_TIMING is on (else -1). */
typedef struct {
    int64_t H, W;
    int64_t n_rd;            /* pixels in RD (label 2) */
    int64_t n_tiles;         /* 32x32 tiles covering the image */
    int64_t n_active_tiles;  /* tiles containing an RD pixel */
    int64_t n_items;         /* strip x 8-row band cells covering the image */
    int64_t n_active_items;  /* stencil work items launched (runs of active cells, split) */
    int64_t n_active_cells;  /* strip x 8-row band cells holding an RD pixel */
    int32_t iters;           /* K of the last solve */
    int32_t k_fuse;          /* iterations fused per HBM round trip */
    int32_t launches;        /* stencil launches in the K-loop */
    int32_t item_rows;       /* maximum output rows per work item (chosen per solve) */
    int32_t item_cols;       /* output columns per work item (strip width) */
    int32_t converged;       /* rds_solve_tol: 1 if the stopping rule fired before max_iters */
    float setup_ms;          /* fused fitting/band/init + compaction */
    float loop_ms;           /* the K-loop (all stencil launches) */
    float residual;          /* rds_solve_tol: max(RMS du, RMS dv) at the last check; else -1 */
    int32_t check_every;     /* rds_solve_tol: iterations between checks; 0 for rds_solve */
    int32_t compact;         /* 1 if the last solve ran the compacted RD iteration (RDS_OPT_COMPACT) */
    int32_t wave;            /* 1 if the last solve's K-loop ran as the temporal wavefront (RDS_OPT_WAVE) */
    int32_t resident;        /* 1 if the last solve ran as one resident cluster (RDS_OPT_RESIDENT),
                                2 if resident on the whole GPU (RDS_OPT_GRID), else 0 */
    int32_t persist;         /* 1 if the last solve's K-loop ran as one persistent launch (RDS_OPT_PERSIST) */
    int32_t rdc_decoupled;   /* compact fixed-K solves: RD pixels with no RD neighbour, iterated
                                independently of the grid-barrier kernel (k_rdc_iso); else 0 */
    int32_t rdc_grouped;     /* compact fixed-K solves: coupled RD pixels in connected components of
                                at most 1024 pixels, iterated inside one warp / CTA each
                                (k_rdc_grp, RDS_OPT_RDC_SPLIT = 2); else 0 */
    int32_t rdc_label_rounds; /* label-propagation rounds the grouping ran (k_grp_prop launches;
                                 0 if it was not tried) */
} rds_stats_t;

/* Options (rds_set_option). */
#define RDS_OPT_KFUSE 1      /* iterations per HBM round trip; 0 = library default; allowed
                                values are listed by rds_kfuse_supported */
#define RDS_OPT_ITEM_ROWS 2  /* maximum output rows per stencil work item (rounded up to a
                                multiple of 8); 0 = automatic (makespan model over resident
                                warps, 8..512 rows) */
#define RDS_OPT_TIMING 3     /* 1 = record setup/loop CUDA-event times in rds_stats_t */
#define RDS_OPT_SKIP 4       /* 1 (default) = work only on strip x 8-row band cells that
                                hold an RD pixel; 0 = process every cell (restriction without
                                skipping) */
#define RDS_OPT_GRAPH 5      /* 1 (default) = replay the K-loop as a CUDA graph */
#define RDS_OPT_CTAS_PER_SM 6 /* cap on resident stencil CTAs per SM (0 = occupancy limit);
                                 a tuning/diagnostic knob, results are identical */
#define RDS_OPT_STOP_NORM 7  /* norm of the stopping rule (rds_solve_tol, rds_solve_gt):
                                0 (default) = Euclidean norm over pixels of unit area,
                                sqrt(sum d^2); 1 = RMS, sqrt(sum d^2 / (H W)) */

#define RDS_OPT_COMPACT 8    /* f3: iterate on the RD pixels alone, stored compactly
                                in row-major RD order with their stencil neighbours' indices, in
                                one persistent cooperative kernel (k_rdc.cu) instead of the dense
                                temporally blocked stencil.  0 = dense; 1 = compact for every
                                rds_solve / rds_solve_q / rds_solve_tol; 2 (default) = compact
                                where a cost model predicts it at least 10% faster (thin
                                scattered bands, e.g. C3 up to delta ~ 0.1 max|f|, and small
                                images), or -- fixed-K solves with RDS_OPT_RDC_SPLIT = 2 -- where
                                the RD density in the active tiles is at most 0.18 and every
                                coupled RD pixel ends up in a grouped component (the compact
                                form is built to find out; if not, the solve runs dense).
                                Same float operations per
                                pixel as the dense path (results agree value for value); the
                                solve synchronises once to size the compact arrays; tolerance
                                solves (rds_solve_tol) evaluate the stopping rule inside the
                                same persistent kernel; images of more than 2^30 pixels and bands
                                of 2^26 or more pixels stay dense. */

#define RDS_OPT_WAVE 9       /* temporal wavefront for fixed-K solves (rds_solve, rds_solve_q,
                                rds_solve_continue): the K / k_fuse blocks of k_fuse fused
                                iterations run as ONE persistent launch in which block b of a
                                column strip follows block b-1 down the image a few rows behind,
                                reading its rows from L2 (progress counters per block and strip;
                                DESIGN.md §5).  Same per-pixel operations as the launch-per-block
                                form: results are bit-identical.  0 = off; 1 = on whenever it
                                applies (image widths a multiple of 4, k_fuse 4..7, at least two
                                full blocks); 2 = on for images above 2^21 pixels.  Default 0:
                                measured slower than the launch-per-block form on B200 (C3
                                25.6 vs 16.5 ms, C4 352 vs 268 ms per 1000 iterations; the
                                chained blocks settle into lock-step polls and the data does not
                                stay in L2).  With no RDS_OPT_KFUSE set it runs
                                k_fuse 6. */

#define RDS_OPT_RESIDENT 10  /* small images (the paper's 128 x 128 size) as ONE resident thread-
                                block cluster: the image in <= 16 horizontal slabs, one CTA each,
                                the state in shared memory, every iteration of a fixed-K solve in
                                one launch with one cluster barrier per iteration (k_small.cu,
                                DESIGN.md §5).  Same per-pixel operations as the stencil (results
                                bit-identical).  Used for rds_solve / rds_solve_q when the slabs
                                fit 200 KB of shared memory per CTA (about 300 x 300 pixels) and
                                the cluster can be scheduled; tolerance solves stay on the
                                stencil.  0 = off; 1 and 2 (default) = on where it applies. */

#define RDS_OPT_PERSIST 11   /* the K-loop of a fixed-K solve as ONE persistent launch of the
                                stencil (k_loop.cu): the K / k_fuse blocks run inside one
                                cooperative grid separated by a grid barrier (or, for <= 16
                                CTAs, the hardware cluster barrier) instead of one launch each;
                                the remainder K mod k_fuse runs as one ordinary launch before.
                                Same per-pixel operations (bit-identical results).  0 (default)
                                = off, 1 = on where it applies (image widths a multiple of 4,
                                k_fuse 4..7, at least two full blocks), 2 = on for images up to
                                2^22 pixels.  Off by default: on B200 the launches are not what
                                bounds these sizes (C0 0.44 vs 0.46 ms, 256^2..2048^2 2-6%
                                slower; the item march's row latency is). */

#define RDS_OPT_GRID 12      /* mid-size images (up to 1024 columns and 8 x #SM rows: C1's
                                1024 x 1024) resident on the whole GPU: every iteration of a
                                fixed-K solve in ONE cooperative launch, the image in G <= #SM
                                horizontal slabs of R <= 8 rows, one CTA per SM, the state in
                                registers, the slab halos exchanged every iteration through an L2
                                mailbox of {value, tag} words that each thread polls for its own
                                columns (no grid barrier, no fence; k_grid.cu).
                                Same per-pixel operations as the stencil (results bit-identical).
                                Applies to rds_solve / rds_solve_q when the resident cluster
                                (RDS_OPT_RESIDENT) does not and the G CTAs can be co-resident;
                                tolerance solves stay on the stencil.  0 (default) = off, 1 and
                                2 = on where it applies.  Off by default: measured on B200 the
                                per-iteration exchange (~1 us) plus the barrier-separated short
                                phases make it slower than the stencil at C1 (3.9 vs 3.0 us per
                                iteration). */

#define RDS_OPT_WS 13        /* warp-specialised stencil (k_stencil_ws.cu): the S-stage pipeline of
                                a full-depth iterating launch split into 2-3-stage chains run by
                                different warps of a CTA, joined through shared-memory hand-off
                                slots one row step apart (the same one-row delay the single-warp
                                kernel's chain split has), so each warp holds 2-3 stages of state
                                and 3-5 CTAs share an SM.  Same per-pixel operations (results
                                bit-identical).  0 (default) = off, 1 = on for image widths a
                                multiple of 4 and k_fuse 6..8.  Off by default: measured on B200
                                it is slower (C3 K-loop 21-25 ms vs 16.3 ms): each warp's one
                                chain is a serial dependency chain, and 3-4 such warps per SM
                                sub-partition hide less latency than 2 warps that interleave
                                three independent chains each. */

#define RDS_OPT_PROLOGUE 14  /* the iterating stencil launches in their prologue form: the first
                                2k+4 row steps of every work item as straight-line code in which
                                the stages still above their dependency cone are elided (6-7% of
                                the stage-rows at k_fuse 7, more for short items).  Same values
                                (bit-identical).  0 = off, 1 = on, 2 (default) = on for images of
                                at most 2^22 pixels, where items are short (C1 -8.6%); off above,
                                where the larger kernel measured no gain. */

#define RDS_OPT_RDC_SPLIT 15 /* compact fixed-K solves (RDS_OPT_COMPACT): RD pixels none of whose six
                                stencil neighbours is RD read no other record and are read by
                                none (the neighbour relation is symmetric), so they iterate as
                                independent threads with the record in registers (k_rdc_iso) and
                                only the coupled rest pays the grid barrier per pass.  2 (default)
                                also finds the connected components of the coupled pixels
                                (an edge wherever one pixel's update reads another's record):
                                a component of at most 1024 pixels runs all K passes inside one
                                warp (<= 32 pixels) or CTA, its records exchanged through shared
                                memory (k_rdc_grp); only larger components keep the grid
                                barrier.  Same values (bit-identical) at every setting.
                                0 = off, 1 = decoupled pixels only, 2 = both. */

/* Create a solver for an H x W image; allocates all device state on the current device.
 * Errors: RDS_EINVAL if out == NULL, H < 1, W < 1 or H*W > 2^31; RDS_ENOMEM / RDS_ECUDA. */
int rds_create(int64_t H, int64_t W, rds_t **out);

/* A batch of B independent H x W images solved together (serving many small images, e.g.
 * the paper's 128 x 128 ones, in one launch sequence).  Inside, image b occupies columns
 * [b W, (b+1) W) of one H x (B W) problem -- narrow images share the stencil's 112-column
 * strips -- and every image keeps its own Neumann last column (grad_2 = 0 on columns W-1,
 * 2W-1, ...), so rho never couples two images.  Every other call takes and returns dense
 * B x H x W buffers (the library transposes to and from its layout); delta, q and the
 * energies apply to the whole batch (energies are sums over the images); active-tile
 * indices refer to the internal H x (B W) layout.  Errors: RDS_EINVAL if B, H or W < 1. */
int rds_create_batch(int64_t B, int64_t H, int64_t W, rds_t **out);

/* Free everything; NULL is a no-op.  Synchronises the handle's stream first. */
int rds_destroy(rds_t *h);

/* All later work is ordered on `stream` (a cudaStream_t, e.g.
 * torch.cuda.current_stream().cuda_stream).  NULL selects the handle's private stream; the
 * legacy default stream is cudaStreamLegacy ((cudaStream_t)0x1) -- the Python binding maps
 * torch's default stream (cuda_stream == 0) to it. */
int rds_set_stream(rds_t *h, void *stream);

/* Set an option (RDS_OPT_*). RDS_EINVAL on unknown key or unsupported value. */
int rds_set_option(rds_t *h, int key, int64_t value);

/* Copy the image z (H x W float32).  Synchronous; checks finiteness.
 * Errors: RDS_EINVAL on NULL or any non-finite value. */
int rds_set_image(rds_t *h, const float *z, int on_device);

/* Fitting constants and the selection map P (H x W float32; may be NULL iff
 * gamma == 0).  Errors: RDS_EINVAL if c1 == c2, gamma < 0 or not finite, P == NULL with
 * gamma > 0, or P non-finite. */
int rds_set_fitting(rds_t *h, float c1, float c2, float gamma, const float *P, int on_device);

/* Optional warm start for the NEXT rds_solve only: v, rho1, rho2 (H x W float32 each).  Used
 * on RD pixels; pinned pixels still start at u0 / 0; rho1 on the last row and rho2 on the last
 * column are zeroed (they are identically 0 under the iteration).  Errors: RDS_EINVAL on NULL. */
int rds_set_state(rds_t *h, const float *v, const float *rho1, const float *rho2,
                  int on_device);

/* Exact float32 max |f| of the current image/fitting (for delta = delta_rel * max|f|).
 * Errors: RDS_ESTATE if image or fitting unset; RDS_EINVAL on NULL. Synchronous. */
int rds_fitting_absmax(rds_t *h, float *out);

/* The q -> q^ search of PAPER.md:74-84 (§3): "q^ is initially 0 and is increased until the
 * selected value of q is satisfied".  Writes the smallest float32 delta such that the band
 * RD = {|f| < delta} holds at least ceil(q * H * W) pixels (pixels tied at the k-th smallest
 * |f| all join RD): delta = nextafter(k-th smallest |f|, +inf); q = 0 gives 0
 * (RD empty, pure thresholding), q = 1 makes every pixel RD.  Exact (4-pass radix select on
 * the bit patterns of |f|, integer histograms); synchronous.
 * Errors: RDS_EINVAL if q not in [0, 1] or delta_out NULL; RDS_ESTATE if image/fitting unset. */
int rds_band_for_fraction(rds_t *h, double q, float *delta_out);

/* rds_band_for_fraction(q) followed by rds_solve with that delta (the paper's control knob). */
int rds_solve_q(rds_t *h, float lambda, float theta, float tau, double q, int32_t iters);

/* Run the whole method: fused fitting + band test + init, active-tile compaction, `iters`
 * outer iterations (rho-step, u-step, v-step) over the active work items, and the output
 * u = v_{K-1} - theta div rho_K on RD (u0 elsewhere) with its mask.  delta is the absolute
 * band threshold (INFINITY = unrestricted, 0 = pure thresholding); iters = 0 yields u = H(-f).
 * Asynchronous on the handle's stream.
 * Errors: RDS_EINVAL if lambda <= 0, theta <= 0, tau not in (0, 1/8], delta < 0 or NaN,
 * iters < 0, or any parameter non-finite (delta may be +inf); RDS_ESTATE if image or fitting
 * unset. */
int rds_solve(rds_t *h, float lambda, float theta, float tau, float delta, int32_t iters);

/* rds_solve with the paper's stopping rule (§4): "iterate until
 *     max{ ||u^(l) - u^(l-1)||, ||v^(l) - v^(l-1)|| } <= delta_stop
 * is met at the l-th iteration".  The norm is the Euclidean norm over all H x W pixels of
 * unit area, like the paper's E2 (reading R-F2; RDS_OPT_STOP_NORM = 1 selects the
 * RMS); pinned pixels contribute 0.  The rule is evaluated after iterations
 * check_every, 2 check_every, ... and always at max_iters (check_every = 0 selects
 * 5 x the library's k_fuse: checking after every launch costs +19% at C3, every 5th
 * +4%); the solve stops at the first check where it holds, else at max_iters.
 * The check runs inside the fused stencil (the launch ending at a check also writes u and
 * the mask) and a one-CTA reduction on the device that also drives a CUDA-graph while loop
 * over whole check blocks, so the call returns without synchronising and the GPU runs only
 * the iterations up to the stop.  The outcome -- iterations
 * done, converged flag, final residual -- is read by rds_get_stats (any getter resolves it).
 * Errors: those of rds_solve, and RDS_EINVAL if tol < 0 or NaN, check_every < 0 or
 * max_iters < 1. */
int rds_solve_tol(rds_t *h, float lambda, float theta, float tau, float delta,
                  int32_t max_iters, float tol, int32_t check_every);

/* ---- float64 mode: the paper's evaluation protocol (§4) ---------------
 * "For delta = 10^-10 we set u^GT(x) = u^(l) in the original dual formulation": a tolerance
 * far below float32 resolution, so rds_solve_gt runs the same iteration (same band test,
 * same stopping rule and RMS norm as rds_solve_tol) with every state array in float64,
 * correctly rounded sqrt/division and no FMA contraction, into separate double planes (the
 * float result of the last rds_solve / rds_solve_tol is untouched).  delta = INFINITY gives
 * the unrestricted ("original") method.  Synchronous.  Errors: as rds_solve_tol, and
 * RDS_EINVAL if check_every < 1. */
typedef struct {
    int32_t iters;      /* iterations done */
    int32_t converged;  /* 1 if the stopping rule fired before max_iters */
    double residual;    /* max(RMS du, RMS dv) at the last check */
} rds_gt_t;
int rds_solve_gt(rds_t *h, float lambda, float theta, float tau, float delta,
                 int32_t max_iters, double tol, int32_t check_every, rds_gt_t *out);

/* u of the last rds_solve_gt, H x W float64.  RDS_ESTATE if none ran. */
int rds_get_u_gt(rds_t *h, double *out, int on_device);

/* The paper's two error measures of the current float u (last rds_solve / rds_solve_tol)
 * against u^GT (last rds_solve_gt), PAPER.md:247-251:
 *   E1 = N(GT n Omega*) / N(GT u Omega*)   (Tanimoto; GT = [u^GT > eps], Omega* = [u > eps];
 *                                           1 when both are empty, reading R-C15)
 *   E2 = sum_x (u(x) - u^GT(x))^2          (unit pixel area, reading R-C15)
 * eps = 0.5 is the paper's convention.  RDS_ESTATE unless both solves ran. */
int rds_compare_gt(rds_t *h, float eps, double *e1, double *e2);

/* Getters: copy H x W results into `out` (host copies synchronise the handle's stream).
 * Errors: RDS_ESTATE before the first solve; RDS_EINVAL on NULL. */
int rds_get_u(rds_t *h, float *out, int on_device);          /* u_K */
int rds_get_mask(rds_t *h, uint8_t *out, int on_device);     /* [u_K > 0.5] as 0/1 */
int rds_get_v(rds_t *h, float *out, int on_device);          /* v_K */
int rds_get_p(rds_t *h, float *rho1, float *rho2, int on_device); /* rho_K */
int rds_get_fitting(rds_t *h, float *out, int on_device);    /* f of the last solve */
int rds_get_labels(rds_t *h, uint8_t *out, int on_device);   /* RDS_LABEL_* per pixel */

/* Ascending list of active tile indices t = ti * ceil(W/tw) + tj (a tile is active iff it
 * contains an RD pixel).  *count always receives the number of active tiles; RDS_EINVAL if
 * cap < count (nothing written then) or count == NULL.  Synchronous. */
int rds_get_active_tiles(rds_t *h, int32_t *out, int64_t cap, int64_t *count);

/* Tile shape used by rds_get_active_tiles (RDS_TILE_H x RDS_TILE_W). */
int rds_tile_shape(int *th, int *tw);

/* Energies of the current (v, rho, u) with the lambda of the last solve (see rds_energy_t).
 * Deterministic two-pass reduction; synchronous.  Errors: RDS_ESTATE before a solve. */
int rds_energy(rds_t *h, rds_energy_t *out);

/* ---- row strips: one image split across ranks ("extension") ----
 * The iteration's dependency cone (rows -2..+1 per iteration, §8(a) S4-S6) lets a handle that
 * holds a row strip of the image plus halo rows reproduce the whole-image iterates exactly on
 * its owned rows: with s iterations between halo refreshes, the rows next to a strip's cut go
 * wrong by at most 2s rows below a top cut and s rows above a bottom cut, so a top halo of
 * >= 2s rows and a bottom halo of >= s + 1 rows keep every owned row (and the row just past
 * it) bit-identical to a whole-image solve, per pixel the same float operations.  The host
 * protocol (paper_1807_11534_b200/strips.py): rds_solve(s) on every strip, then repeatedly
 * exchange halo rows (rds_get_state_rows -> neighbour's rds_set_state_rows) and
 * rds_solve_continue(s).  delta must be the same absolute value on every strip. */

/* Run `iters` more iterations from the current state with the parameters, labels and work
 * items of the last rds_solve / rds_solve_tol / rds_solve_q (no setup; fixed K; writes u and
 * the mask at the end).  A tolerance solve's outcome is resolved first (synchronises).
 * iters = 0 is a no-op.  Errors: RDS_ESTATE before a solve; RDS_EINVAL if iters < 0. */
int rds_solve_continue(rds_t *h, int32_t iters);

/* rds_solve_continue(iters) whose last iteration l also evaluates the two sums of the paper's
 * stopping rule (§4) over rows [row0, row1) only:
 *   sums[0] = sum (u^l - u^(l-1))^2,  sums[1] = sum (v^l - v^(l-1))^2   (host, synchronises).
 * A strip passes its owned rows; the ranks all-reduce the sums and take one decision, so the
 * rule runs on a strip-decomposed image exactly as on the whole one (strips.StripSolver.
 * solve_tol).  Errors: RDS_ESTATE before a solve; RDS_EINVAL if iters < 1, sums == NULL or the
 * rows leave [0, H). */
int rds_continue_check(rds_t *h, int32_t iters, int64_t row0, int64_t row1, double *sums);

/* One radix-select pass of rds_band_for_fraction over rows [row0, row1): out[d] (256 counts,
 * host) = #{pixels of those rows whose |f| bit pattern b has (b & mask) == prefix and byte
 * (b >> shift) & 255 == d}, shift in {24, 16, 8, 0}.  |f| >= 0, so bit patterns order like
 * the values; summing the strips' histograms (all-reduce) and walking the passes from the
 * top byte down finds the k-th smallest |f| of the whole image (the q -> q^ rule of
 * PAPER.md:74, 84; strips.StripSolver.band_for_fraction).  Synchronises.  Errors:
 * RDS_ESTATE before rds_set_image / rds_set_fitting; RDS_EINVAL on NULL, rows outside
 * [0, H) or another shift. */
int rds_abs_histogram(rds_t *h, int64_t row0, int64_t row1, uint32_t prefix, uint32_t mask,
                      int32_t shift, uint32_t *out);

/* Copy rows [row0, row0 + nrows) of the current state out of / into the handle.  Buffer
 * layout: three planes v, rho1, rho2, each nrows x W float32 row-major (natural column
 * order), i.e. 3 * nrows * W floats.  Host buffers (on_device = 0) are synchronous; device
 * buffers are stream-ordered.  Setting rows replaces the state the next rds_solve_continue
 * starts from (labels and c' are not touched).  Errors: RDS_ESTATE before a solve;
 * RDS_EINVAL if the rows leave [0, H), nrows < 0, buffer NULL with nrows > 0, or a batch
 * handle. */
int rds_get_state_rows(rds_t *h, int64_t row0, int64_t nrows, float *out, int on_device);
int rds_set_state_rows(rds_t *h, int64_t row0, int64_t nrows, const float *in, int on_device);

/* Rows summed by rds_energy: [row0, row1) (row1 < 0 means H; default all rows).  A strip
 * sums only its owned rows; the terms at the last owned row read the row below it (the
 * halo).  Summing the strips' TV_v, fit_v, E_u and D_p then gives the whole image's.
 * Errors: RDS_EINVAL unless 0 <= row0 <= row1 <= H. */
int rds_set_energy_rows(rds_t *h, int64_t row0, int64_t row1);

/* Statistics of the last solve (synchronises the stream). */
int rds_get_stats(rds_t *h, rds_stats_t *out);

/* Diagnostic (memory safety without a sanitizer): the number of elements in the padded frame
 * around the image, over every device plane, that no longer hold the pinned value they were
 * allocated with (rho = v = u = f = z = 0, c' = +inf, labels = mask = 0).  Any nonzero count
 * means a kernel wrote outside the image.  Synchronous. */
int rds_check_frame(rds_t *h, int64_t *bad_count);

/* Supported RDS_OPT_KFUSE values: writes up to cap values into out, returns how many exist. */
int rds_kfuse_supported(int32_t *out, int cap);

/* Message for the last failure on h ("" if none); h == NULL gives the last global failure
 * (e.g. from rds_create). Valid until the next call on that handle. */
const char *rds_last_error(rds_t *h);

/* Library version string. */
const char *rds_version(void);

/* ---- f4: 3-D volumes (§5 "extension to 3D") -------------------------------
 * The same method on a D x H x W volume (plane-major, row-major planes): voxel labels and
 * fitting term as above; grad = forward differences along rows, columns and planes with a
 * zero last row / column / plane, div = -grad^T, rho = (rho1 rows, rho2 columns, rho3 planes)
 * (reading R-F4).  tau must be in (0, 1/12] (||grad||^2 <= 12 in 3-D).  k_fuse
 * iterations per fused pass over the volume (1, the default: k_vol_step, one pass per
 * iteration; 2-3: k_vol_tb, temporal blocking along the plane axis, measured slower on B200),
 * the K-loop replayed from a CUDA graph.
 * Errors as for the 2-D calls; the buffers are D*H*W elements. */
typedef struct rds3_handle rds3_t;
int rds3_create(int64_t D, int64_t H, int64_t W, rds3_t **out);
int rds3_destroy(rds3_t *h);
int rds3_set_stream(rds3_t *h, void *stream);
/* planes per CTA z-chunk (0 = automatic); a tuning knob, results identical */
int rds3_set_kz(rds3_t *h, int32_t kz);
/* iterations per pass over the volume, 1 .. 3 (0 = automatic: 1); every value gives the same
 * bits (the passes run the same per-voxel operations in the same order); RDS_EINVAL outside */
int rds3_set_kfuse(rds3_t *h, int32_t kf);
int rds3_set_image(rds3_t *h, const float *z, int on_device);
int rds3_set_fitting(rds3_t *h, float c1, float c2, float gamma, const float *P, int on_device);
int rds3_fitting_absmax(rds3_t *h, float *out);
int rds3_solve(rds3_t *h, float lambda, float theta, float tau, float delta, int32_t iters);
int rds3_get_u(rds3_t *h, float *out, int on_device);
int rds3_get_v(rds3_t *h, float *out, int on_device);
int rds3_get_p(rds3_t *h, float *rho1, float *rho2, float *rho3, int on_device);
int rds3_get_mask(rds3_t *h, uint8_t *out, int on_device);
int rds3_get_labels(rds3_t *h, uint8_t *out, int on_device);
/* voxels in RD, K of the last solve, planes per CTA z-chunk, setup + K-loop time (ms) */
int rds3_get_stats(rds3_t *h, int64_t *n_rd, int32_t *iters, int32_t *kz, float *ms);
const char *rds3_last_error(rds3_t *h);

#ifdef __cplusplus
}
#endif

#endif /* RDS_H_ */
