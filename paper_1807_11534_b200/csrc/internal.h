// internal.h -- shared declarations of the librds CUDA product path (not part of the ABI).
//
// Device-memory layout ("padded planes"): every per-pixel array is a plane of
// (H + 2*PAD_R) rows x pitch elements; pixel (i, j) lives at element
//     origin + i * pitch + j,   origin = PAD_R * pitch + PAD_C.
// The frame outside the image holds *pinned background* values (rho = 0, v = 0,
// c = +inf) that the iteration reproduces exactly, so the stencil needs no bounds tests on
// loads: only the two Neumann conditions (grad_1 = 0 on row H-1, grad_2 = 0 on column W-1)
// are explicit.  pitch is a multiple of 32 elements (128 B rows for float planes).
//
// The stencil's state planes (rho1, rho2, v in both ping-pong buffers, and c) are
// QUAD-SWIZZLED: within every aligned quad of columns 4g..4g+3 the memory order is
// x0 x2 x1 x3 (swap of index bits 0 and 1), so one 16-byte load gives the packed f32x2
// pairs (x0, x2), (x1, x3) the stencil computes on (k_stencil_impl.cuh).  PAD_C is a multiple of
// 4, so the swizzle applies to the column index relative to the origin.  z, P, f, u, the
// labels and the mask are natural-order planes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rds {

constexpr int PAD_R = 16;      // >= KF + 1 rows of halo above / below (KF <= 15)
constexpr int PAD_C = 32;      // left frame, keeps column 0 16-byte aligned
constexpr int PAD_C_RIGHT = 128;  // a warp strip may read up to 127 columns past its start
constexpr int TILE_H = 32, TILE_W = 32;
// work-item activity is decided per strip x BAND_H-row band, from RD counts per 32-column x
// BAND_H-row sub-tile (SUBTILES per 32x32 tile)
constexpr int BAND_H = 8, SUBTILES = TILE_H / BAND_H;
constexpr int STENCIL_WARPS = 4;

// element offset of column j inside a quad-swizzled row (valid for negative j as well)
__host__ __device__ constexpr int swz(int j) { return (j & ~3) | ((j & 1) << 1) | ((j >> 1) & 1); }  // warps per CTA of the stencil kernel (one item per warp)

// Column geometry of a stencil warp for KF fused iterations: the warp loads 128 columns
// (float4 per lane); the valid output columns are [LH, LH + WV) of those.  The dependency
// cone of KF iterations reaches KF+1 columns to the left and KF to the right
// (DESIGN.md §5), rounded up to whole float4 lanes.
__host__ __device__ constexpr int lh_of(int kf) { return 4 * ((kf + 1 + 3) / 4); }
__host__ __device__ constexpr int rh_of(int kf) { return 4 * ((kf + 3) / 4); }
__host__ __device__ constexpr int wv_of(int kf) { return 128 - lh_of(kf) - rh_of(kf); }

// The next run [b, e) of set bits at or after position *pos in a strip's band bitmask
// (nbw words); false when there is none.  *pos is left at e.
__device__ __forceinline__ bool next_run(const uint32_t *bits, int nbw, int *pos, int *b, int *e) {
    int p = *pos, w = p >> 5;
    if (w >= nbw) return false;
    uint32_t x = bits[w] & (0xffffffffu << (p & 31));
    while (x == 0) {
        if (++w >= nbw) return false;
        x = bits[w];
    }
    *b = (w << 5) + __ffs(x) - 1;
    // run end: first clear bit after b
    p = *b;
    uint32_t y = ~bits[w] & (0xffffffffu << (p & 31));
    while (y == 0) {
        if (++w >= nbw) {
            *e = nbw << 5;
            *pos = *e;
            return true;
        }
        y = ~bits[w];
    }
    *e = (w << 5) + __ffs(y) - 1;
    *pos = *e;
    return true;
}

// A stencil work item: output columns [strip*WV, (strip+1)*WV) and output rows [r0, r1) --
// a piece of a vertical run of active 32-row bands, cut at multiples of ITEM_Q rows.
constexpr int ITEM_Q = 8;
struct Item {
    int32_t strip, r0, r1, pad_;
};

// Device record of a tolerance solve (rds_solve_tol, rds_solve_gt): written by k_stop_check
// only; zeroed before the solve.
struct StopRecord {
    int32_t flag;       // 1 once the rule fired (or the last check ran): later launches exit
    int32_t iters;      // iterations completed when it fired
    int32_t launches;   // stencil launches that ran (selects the ping-pong buffer)
    int32_t converged;  // residual <= tol at that check
    double residual;    // ||du||, ||dv|| max at the last check (norm: StopCheck::norm_div)
    int32_t checks;     // checks evaluated
    int32_t it;         // iterations done so far (advanced by every check)
    double su, sv;      // the last check's sums of (u^l - u^(l-1))^2, (v^l - v^(l-1))^2
};

// One evaluation of the stopping rule after a block of iterations.
struct StopCheck {
    const double *part;        // [n][2] partial sums of du^2, dv^2
    const int32_t *n_part;     // device count n
    double norm_div;           // 1 = Euclidean norm over pixels, H*W = RMS (reading R-F2)
    double tol;
    int block_iters;           // iterations of the block this check closes
    int block_launches;        // stencil launches of that block (ping-pong parity)
    int max_iters;             // the solve's K: the check at rec->it == K is the last
    int set_cond;              // 1: also drive the enclosing CUDA-graph while loop
    int body_iters;            // iterations per loop body, and the loop's last iteration:
    int loop_end;              //   continue iff !fired && it + body_iters <= loop_end
    cudaGraphConditionalHandle cond;
    StopRecord *rec;
};

struct StencilArgs {
    const float *p1_in, *p2_in, *v_in;   // plane origins (pixel (0,0))
    const float *c;                      // 2^-100 theta*lambda*f on RD, -inf Fg, +inf Bg/frame
    float *p1_out, *p2_out, *v_out;
    float *u_out;                        // only written when WRITE_U
    uint8_t *mask_out;                   // only written when WRITE_U
    const Item *items;                   // active items (strip-major, runs split in chunks)
    const int32_t *n_items;              // device count
    int32_t *queue;                      // this launch's work counter (zeroed before the loop)
    StopRecord *stop;                    // tolerance mode: skip the launch once stop->flag
    double *chk;                         // CHECK launches: [item][2] sums of du^2, dv^2
    int chk_r0, chk_r1;                  // CHECK launches: rows the sums cover ([0, H) for a
                                         // whole-image rule; a strip's owned rows)
    int64_t pitch;
    int H, W;
    int img_w;                           // columns per image (W, or the image width of a batch)
    float tau, theta, inv_theta;
    int ws;                              // full-depth PLAIN launches on k_stencil_ws (RDS_OPT_WS)
    int pro;                             // PLAIN launches in the prologue form (RDS_OPT_PROLOGUE)
};

// The temporal wavefront (k_wave.cu): nblk blocks of KF iterations of a
// fixed-K solve in ONE persistent launch; block b of strip s reads ping-pong buffer
// (c0 + b) & 1 and writes the other, after its producers (block b-1, strips s-1..s+1) have
// published the rows it needs in prog[(b-1) * n_strips + s'] (rows < value final).
struct WaveArgs {
    StencilArgs a;                       // c, pitch, H, W, img_w, tau, theta (planes below)
    const float *p1[2], *p2[2], *v[2];   // ping-pong plane origins
    const uint32_t *band_bits;           // active 8-row bands per strip (launch_band_flags)
    int nbw;                             // bitmask words per strip
    int32_t *prog;                       // [nblk][n_strips], zeroed before the launch
    int32_t *queue;                      // task counter, zeroed before the launch
    int nblk, n_strips, c0;
};
cudaError_t launch_wave(int kf, const WaveArgs &w, int grid, cudaStream_t s);
int wave_blocks_per_sm(int kf);
bool wave_supported(int kf);

// Small images as one resident cluster (k_small.cu): G slabs of R rows, one CTA
// each (one thread per column), the whole fixed-K loop in one launch.  Reads the state from the
// dense ping-pong buffer *_in, writes the final state into *_out and u / the mask of the last
// iteration.
constexpr int SMALL_THREADS_MAX = 1024, SMALL_MAX_CTAS = 16;
struct SmallArgs {
    const float *p1_in, *p2_in, *v_in, *c;   // plane origins (pixel (0,0)), swizzled
    float *p1_out, *p2_out, *v_out;
    float *u_out;
    uint8_t *mask_out;
    const long long *n_rd;                   // RD pixel count (0: nothing moves), or null
    int64_t pitch;
    int H, W, img_w, K, G, R;
    float tau, theta, inv_theta;
};
bool small_plan(int64_t H, int64_t W, int *G, int *R);
bool small_cluster_fits(const SmallArgs &a);
cudaError_t launch_small(const SmallArgs &a, cudaStream_t s);

// Mid-size images resident on the whole GPU (k_grid.cu): G <= #SM slabs of R
// rows, one cooperative CTA each, halos through an L2 mailbox of {value, tag} words.
struct GridArgs {
    const float *p1_in, *p2_in, *v_in, *c;   // plane origins (pixel (0,0)), swizzled
    float *p1_out, *p2_out, *v_out;
    float *u_out;
    uint8_t *mask_out;
    const long long *n_rd;                   // RD pixel count (0: nothing moves), or null
    unsigned long long *mail;                // [2][G][7][2 * threads] {value, tag} words
    unsigned tag0;                           // tag of iteration 0 (grows across launches)
    int64_t pitch;
    int H, W, img_w, K, G, R;
    float tau, theta, inv_theta;
};
bool grid_plan(int64_t H, int64_t W, int n_sm, int *G, int *R);
size_t grid_mail_words(int G, int W);
bool grid_fits(const GridArgs &a);
cudaError_t launch_grid(const GridArgs &a, cudaStream_t s);

// The fixed-K K-loop as one persistent launch (k_loop.cu): nblk blocks of KF
// iterations over the same work items, block b reading ping-pong buffer (c0 + b) & 1, a grid
// (or cluster) barrier between blocks, the last block writing u and the mask.
struct LoopArgs {
    StencilArgs a;                       // c, u / mask, items, n_items, pitch, H, W, img_w, ...
    const float *p1[2], *p2[2], *v[2];   // ping-pong plane origins
    int32_t *queue;                      // [nblk] per-block item counters, zeroed
    unsigned long long *bar;             // grid-barrier counter (zeroed by the launcher)
    int nblk, c0;
};
bool loop_supported(int kf);
int loop_blocks_per_sm(int kf);
cudaError_t launch_loop(int kf, const LoopArgs &L, int grid, cudaStream_t s);

// launchers (return cudaError_t of the launch)
cudaError_t launch_fill_frame(float *plane, int64_t n, float value, cudaStream_t s);
cudaError_t launch_check_finite(const float *a, int64_t pitch, int H, int W, int *flag,
                                cudaStream_t s);
cudaError_t launch_absmax(const float *z, const float *P, int64_t pitch, int H, int W,
                          float c1, float c2, float gamma, unsigned *out_bits,
                          cudaStream_t s);

cudaError_t launch_abs_hist(const float *z, const float *P, int64_t pitch, int H, int W,
                            float c1, float c2, float gamma, unsigned prefix, unsigned mask,
                            int shift, unsigned *hist, cudaStream_t s);

struct SetupArgs {
    const float *z, *P;                 // P may be null when gamma == 0
    const float *wv, *wp1, *wp2;        // warm start (null = none)
    float *f, *c, *u;
    float *v0, *v1, *p10, *p11, *p20, *p21;
    uint8_t *lab, *mask;
    int32_t *tile_rd;                   // RD pixels per 32x32 tile
    int32_t *sub_rd;                    // RD pixels per 32-column x BAND_H-row sub-tile
    int64_t pitch;
    int H, W, img_w;
    float c1, c2, gamma, delta, theta_lambda;
};
cudaError_t launch_setup(const SetupArgs &a, cudaStream_t s);

// Deterministic ballot/prefix-sum compaction of flags[i] != 0 into an ascending index list.
// counts[0] = number of nonzero flags; if sum_out != null also the int64 sum of the values.
cudaError_t launch_compact(const int32_t *flags, int n, int32_t *list, int32_t *count,
                           long long *sum_out, cudaStream_t s);
// band_bits[s * ceil(n_bands/32) + b/32] bit b%32 = 1 iff strip s (output columns
// [s*wv, (s+1)*wv)) overlaps an 8-row band b holding an RD pixel (skip = 0: every band).
cudaError_t launch_band_flags(const int32_t *sub_rd, int H, int W, int wv, int n_strips,
                              int skip, uint32_t *band_bits, cudaStream_t s);
// Work items from the band flags: maximal vertical runs of active bands per strip, each split
// into ceil(rows / chunk) near-equal pieces at ITEM_Q-row boundaries.  chunk = fixed_chunk
// rounded up to ITEM_Q if > 0, else the candidate height minimising
// ceil(items / slots) * (chunk + warmup_rows) (makespan model, k_setup.cu).
// out: items, counts[1] = number of items, counts[2] = chunk rows, counts[3] = active cells.
cudaError_t launch_build_items(const uint32_t *band_bits, int n_strips, int n_bands, int H,
                               int slots, int fixed_chunk, int max_chunk, int warmup_rows,
                               Item *items, int32_t *counts, cudaStream_t s);

// mode: 0 iterate, 1 + write u and mask, 2 + stopping sums into a.chk (k_stencil_impl.cuh)
cudaError_t launch_stencil(int kf, int stages, int mode, const StencilArgs &a,
                           int grid, cudaStream_t s);
int stencil_blocks_per_sm(int kf, int stages, bool aligned);
// concurrent stencil workers per SM for full-depth launches (warps, or CTAs of k_stencil_ws)
int stencil_workers_per_sm(int kf, bool aligned, bool ws);
// k_stencil_ws.cu: warp-specialised stage chains (MODE_PLAIN, aligned, stages == k_fuse)
bool ws_available(int stages);
int ws_blocks_per_sm(int stages);
cudaError_t launch_stencil_ws(int stages, const StencilArgs &a, int grid, cudaStream_t s);
bool kf_supported(int kf);
int kf_list(int32_t *out, int cap);
// Stopping rule after a block of iterations (k_energy.cu).
cudaError_t launch_stop_check(const StopCheck &c, cudaStream_t s);

struct EnergyArgs {
    const float *f, *u, *v, *p1, *p2;
    const uint8_t *lab;           // labels (F^RD: the sum over RD and u0 off RD)
    int64_t pitch;
    int H, W, img_w;
    int row0, row1;     // rows summed: [row0, row1) (rds_set_energy_rows; default [0, H))
    double *partials;   // [n_blocks * 7]
    double *out;        // [7]: TV_v, sum f v, TV_cu, sum f cu, sum min(0, lambda f + div p),
                        //      sum_RD |grad u'|, sum (u' - v)^2
    float lambda, theta;
};
constexpr int ENERGY_BLOCKS = 592;  // 4 x 148 SMs (k_energy_partial)
constexpr int ENERGY_WARPS = 8192;  // bound on k_energy_strip's warps (its partials)
cudaError_t launch_energy(const EnergyArgs &a, cudaStream_t s);

// f3: compacted restricted-domain iteration (k_rdc.cu).  Neighbour codes: >= 0 compact index
// of an RD pixel; RDC_BG / RDC_FG a pinned pixel (rho = 0, v = u0 = 0 / 1) or the frame;
// RDC_EDGE the missing forward neighbour on row H-1 / an image's last column (grad = 0).
constexpr int RDC_BG = -1, RDC_FG = -2, RDC_EDGE = -3;
// Packed neighbour codes, two words per RD pixel: word A = the RD index of (i-1, j), else of
// (i-1, j+1) | classes of up, up-right, left << RDC_IDX_BITS; word B = the RD index of
// (i+1, j), else of (i+1, j-1) | classes of down, down-left, right.  2-bit classes:
constexpr unsigned RDC_C_RD = 0, RDC_C_BG = 1, RDC_C_FG = 2, RDC_C_EDGE = 3;
constexpr int RDC_IDX_BITS = 26;  // compact path only for n_rd < 2^26
constexpr unsigned RDC_IDX_MASK = (1u << RDC_IDX_BITS) - 1u;
__host__ __device__ inline unsigned rdc_cls(int code) {
    return code >= 0 ? RDC_C_RD : (code == RDC_FG ? RDC_C_FG : (code == RDC_EDGE ? RDC_C_EDGE : RDC_C_BG));
}
constexpr int RDC_MAX_GRID = 4 * 148 * 4;  // bound on k_rdc_iter CTAs (the stopping-sum buffer)
// grid barrier counter (one 128-byte line), then the per-CTA pass counters of the neighbour
// synchronisation (k_rdc_iter NB form)
constexpr int RDC_BAR_BYTES = 128 + 4 * RDC_MAX_GRID;
constexpr int RDC_THREADS = 512;
constexpr int RDC_CLUSTER_MAX = 16;  // CTAs of the one-cluster form (non-portable size)
struct RdcSetup {
    int n, H, W, img_w;
    int64_t pitch;
    const int32_t *list, *idxmap;
    uint2 *code;                  // packed neighbour codes
    float4 *rec;                  // (rho1, rho2, v, c') per RD pixel (gather: start; scatter: final)
    float *u;
    const float *cplane;          // dense plane origins
    float *p1plane, *p2plane, *vplane, *uplane;
    uint8_t *mask;
};
struct RdcIter {
    int n, K;
    const uint2 *code;
    float4 *rec[2];               // pass k reads rec[k & 1], writes rec[(k + 1) & 1]
    float *u;
    float tau, theta, inv_theta;
    unsigned long long *bar;      // RDC_BAR_BYTES, zeroed per launch (64-bit: never wraps)
    // tolerance solves (check_every > 0): per-CTA partial sums, the outcome (StopRecord
    // fields iters, converged, residual, checks, flag; launches = 0)
    int check_every;
    double tol, norm_div;
    double *part;                 // [2][2 * RDC_MAX_GRID]: alternate by check parity (a fast
                                  // CTA's next check must not overwrite sums still being read)
    StopRecord *rec_out;
    const int32_t *sel;           // split solves: the n coupled record indices (else null: 0..n-1)
};
cudaError_t launch_rdc_count(const uint8_t *lab, int64_t pitch, int H, int W, int32_t *rowcnt,
                             int32_t *rowoff, int32_t *total, cudaStream_t s);
cudaError_t launch_rdc_fill(const uint8_t *lab, int64_t pitch, int H, int W,
                            const int32_t *rowoff, int32_t *idxmap, int32_t *list,
                            cudaStream_t s);
cudaError_t launch_rdc_gather(const RdcSetup &a, cudaStream_t s);
cudaError_t launch_rdc_scatter(const RdcSetup &a, const RdcIter &it, cudaStream_t s);
cudaError_t launch_rdc_iter(const RdcIter &a, int n_sm, cudaStream_t s);
// split of the n records into coupled (cpl, ascending) and decoupled ones (iso, ascending);
// cnt / off: ceil(n / 1024) + 1 ints each, *n_cpl: the coupled count
cudaError_t launch_rdc_split(const uint2 *code, int n, int32_t *cnt, int32_t *off,
                             int32_t *n_cpl, int32_t *cpl, int32_t *iso, cudaStream_t s);
// the K passes of the n_iso decoupled records (fixed-K solves), independent of the barrier kernel
cudaError_t launch_rdc_iso(const RdcIter &a, const int32_t *iso, int n_iso, int n_sm,
                           cudaStream_t s);

// grouped coupled records (RDS_OPT_RDC_SPLIT = 2, k_rdc.cu): connected components of the
// coupled list that fit one warp / CTA iterate there; the rest is the fallback list
struct GrpPlan {
    int base[11] = {};   // first slot of class k (slot range 2^k, k = 1 .. 10)
    int first[3] = {};   // first slot of segment 0 (warp blocks), 1 (256), 2 (1024)
    int count[3] = {};   // slots in use per segment
    int total = 0;       // slots allocated (segments padded to multiples of 1024)
    int rounds = 0;      // label rounds run (k_grp_prop launches)
};
// labels, per-label counts / flags, per-record ranks, per-root class and index; ctr: 16 ints
// (ctr[k] = components of class k = 1 .. 10, ctr[11] = grouped records)
cudaError_t launch_grp_label(const uint2 *code, const int32_t *cpl, int nc, int32_t *lab,
                             int32_t *cnt, int32_t *bad, int32_t *rank, int32_t *cidx,
                             int32_t *ctr, int *rounds, cudaStream_t s);
void grp_layout(const int32_t *ctr, GrpPlan *gp);
cudaError_t launch_grp_fill(const int32_t *cpl, int nc, const int32_t *lab, const int32_t *cidx,
                            const int32_t *rank, const GrpPlan &gp, int32_t *slots,
                            int32_t *lpos, int32_t *fb, int32_t *nfb, cudaStream_t s);
cudaError_t launch_rdc_grp(const RdcIter &a, const GrpPlan &gp, const int32_t *slots,
                           const int32_t *lpos, cudaStream_t s);

// float64 mode (k_fp64.cu): natural-order padded double planes, same pitch as the floats
struct F64Args {
    const float *z, *P;        // image and selection map (float planes; P may be null)
    double *f, *u, *v;
    double *v2;                // second v buffer of the persistent solve (k64_persist), or null
    double *p1[2], *p2[2];     // ping-pong rho
    uint8_t *lab;
    StopRecord *stop;          // outcome of the tolerance solve
    int64_t pitch;
    int H, W, img_w;
    float c1, c2, gamma, delta;
    double tau, theta, theta_lambda;
};
constexpr int F64_BLOCKS = 592;  // fixed grid of the double-precision kernels (4 x 148)
int f64_grid(int64_t n);
cudaError_t launch_f64_init(const F64Args &a, cudaStream_t s);
// the whole fp64 tolerance solve as one cooperative launch (k64_persist)
constexpr int F64P_THREADS = 256, F64P_MAX_GRID = 4 * 148 * 4;
struct F64Persist {
    F64Args a;                 // a.v = v buffer 0 (v^0 after init), a.stop = the outcome
    double *v[2];
    int max_iters, check_every;
    double tol, norm_div;
    double *part;              // [2][2 * F64P_MAX_GRID], alternating by check parity
    unsigned long long *bar;   // 64-bit barrier counter (no wrap at any max_iters)
};
cudaError_t launch_f64_persist(const F64Persist &q, int n_sm, cudaStream_t s);
// E1, E2 of the float u against a double u (out[0], out[1]); part holds 3 doubles per CTA
cudaError_t launch_compare(const float *u, const double *ugt, int64_t pitch, int H, int W,
                           float eps, double *part, double *out, cudaStream_t s);

// f4: 3-D volumes (k_vol.cu).  Padded volume: VOL_PZ frame planes before/after, VOL_PY_TOP
// rows above and VOL_PY_BOT below each plane, VOL_PX_L columns left, >= VOL_PX_R right.
constexpr int VOL_PZ = 4, VOL_PY_TOP = 8, VOL_PY_BOT = 32, VOL_PX_L = 8, VOL_PX_R = 32;
constexpr int VOL_TB_MAX = 3, VOL_TB_DEFAULT = 1;  // k_vol_tb measured slower on B200  // iterations per pass of k_vol_tb (frame: VOL_PZ >= S + 1, 2S rows / columns)
struct VolArgs {
    const float *p1_in, *p2_in, *p3_in, *v_in, *c;   // voxel (0,0,0) origins
    float *p1_out, *p2_out, *p3_out, *v_out, *u_out;
    uint8_t *mask_out;
    int64_t plane, pitch;
    int D, H, W, kz;                                 // kz = planes per CTA z-chunk
    float tau, theta, inv_theta;
};
struct VolSetupArgs {
    const float *z, *P;
    float *f, *c, *u, *v0, *v1, *p10, *p11, *p20, *p21, *p30, *p31;
    uint8_t *lab, *mask;
    unsigned long long *n_rd;
    int64_t plane, pitch;
    int D, H, W;
    float c1, c2, gamma, delta, theta_lambda;
};
cudaError_t launch_vol_step(const VolArgs &a, bool write_u, cudaStream_t s);
int64_t vol_tiles(int64_t H, int64_t W);  // CTA (i, j) tiles of k_vol_step
// S iterations per pass (k_vol_tb, S = 1 .. VOL_TB_MAX): launch, (i, j) tiles, CTAs per SM
cudaError_t launch_vol_tb(const VolArgs &a, int S, bool write_u, cudaStream_t s);
int64_t vol_tb_tiles(int S, int64_t H, int64_t W);
int vol_tb_blocks_per_sm(int S);
cudaError_t launch_vol_setup(const VolSetupArgs &a, cudaStream_t s);
cudaError_t launch_vol_absmax(const float *z, const float *P, int64_t plane, int64_t pitch,
                              int D, int H, int W, float c1, float c2, float gamma,
                              unsigned *out_bits, cudaStream_t s);
cudaError_t launch_vol_copy_f32(float *dst, const float *src, int64_t plane, int64_t pitch,
                                int D, int H, int W, int to_padded, cudaStream_t s);
cudaError_t launch_vol_copy_u8(uint8_t *dst, const uint8_t *src, int64_t plane, int64_t pitch,
                               int D, int H, int W, int to_padded, cudaStream_t s);

// out[i * out_pitch + j] = plane[i * pitch + swz(j)]: natural-order copy of a swizzled plane
cudaError_t launch_unswizzle(const float *plane, int64_t pitch, int H, int W, float *out,
                             int64_t out_pitch, cudaStream_t s);
// Count frame elements of a padded plane that no longer hold their pinned value.
cudaError_t launch_frame_check(const void *base, int elt, int64_t pitch, int64_t rows,
                               int64_t origin_row, int64_t origin_col, int H, int W,
                               int swizzled, double expect, unsigned long long *bad,
                               cudaStream_t s);
// Batch layout (rds_create_batch): image b of B (H x img_w each) occupies columns
// [b img_w, (b+1) img_w) of the H x (B img_w) planes.  Dense (B, H, img_w) <-> plane copies
// (elt = 8, 4 or 1 bytes; swizzled = the plane is quad-swizzled, for rho and v).
cudaError_t launch_batch_copy(void *dense, void *plane, int elt, int64_t pitch, int H,
                              int img_w, int B, int to_plane, int swizzled, cudaStream_t s);

}  // namespace rds
