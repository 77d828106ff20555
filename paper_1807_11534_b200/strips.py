"""Row strips: one image split across ranks (§5, names larger
problems as the method's extension).

Every iteration of Eq. 7-9 reads, for the new state at row i, the old
state at rows i-2 .. i+1 (SURVEY §8(a) S4-S6 footprint).  A handle that holds a strip of rows
plus halo rows therefore computes its owned rows exactly as a whole-image solve would, as
long as the rows it got wrong at its cuts (the strip's first row lacks the row above it, its
last row the row below) have not reached them: after s iterations the damage reaches 2s rows
down from a top cut and s rows up from a bottom cut.  With a top halo of 2s rows and a bottom
halo of s + 1 rows, refreshed from the neighbours every s iterations, the owned rows and the
row just below them stay bit-identical to the whole-image iterates (same float operations per
pixel), which is what `tests/test_gpu_strips.py` checks on one GPU and
`tests/test_dist_cpu.py` checks for the torch.distributed exchange with the CPU oracle.

The exchange is the path's one real communication step: per refresh each cut moves
(2s + s + 1) rows x W x (v, rho1, rho2) float32, e.g. 22 rows x 16384 x 12 B = 4.3 MB at
C4 with s = 7, against 7 iterations of ~34 M pixels per GPU at G = 8.  It uses
torch.distributed point-to-point (NCCL on GPUs; gloo on CPU for the tests) on the handle's
stream (torch's current stream).  Everything else a strip needs is rank-local; delta must be
the same absolute value everywhere (`absmax` all-reduces max |f|) and energies are summed
over ranks (`energy`).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def halo_rows(seg_iters: int) -> tuple[int, int]:
    """(top, bottom) halo rows for `seg_iters` iterations between refreshes."""
    if seg_iters < 1:
        raise ValueError("seg_iters must be >= 1")
    return 2 * seg_iters, seg_iters + 1


@dataclass(frozen=True)
class Strip:
    rank: int
    lo: int     # owned global rows [lo, hi)
    hi: int
    top: int    # halo rows held above lo / below hi
    bot: int

    @property
    def r0(self) -> int:  # first global row held
        return self.lo - self.top

    @property
    def rows(self) -> int:  # rows held
        return self.hi - self.lo + self.top + self.bot

    @property
    def owned(self) -> slice:  # owned rows in local coordinates
        return slice(self.top, self.top + self.hi - self.lo)


def partition(H: int, G: int, seg_iters: int, weights=None) -> list[Strip]:
    """G row strips of an H-row image, each with the halos of `halo_rows(seg_iters)` (none at
    the image's own top and bottom).  Without `weights`: near-equal strips (the first H % G
    one row taller).  With `weights` (H non-negative per-row costs, e.g. `row_weights` of the
    band labels): the cuts balance the owned rows' total weight -- a restricted solve costs
    what its active rows cost, not its row count -- under the constraint that
    every strip owns at least the top-halo rows its neighbour below needs."""
    if G < 1 or H < G:
        raise ValueError(f"cannot split {H} rows into {G} strips")
    top, bot = halo_rows(seg_iters)
    if weights is None:
        base, extra = divmod(H, G)
        cuts = [0]
        for k in range(G):
            cuts.append(cuts[-1] + base + (1 if k < extra else 0))
    else:
        cuts = _weighted_cuts(np.asarray(weights, dtype=np.float64), G,
                              max(1, top) if G > 1 else 1)
    out = []
    for k in range(G):
        out.append(Strip(k, cuts[k], cuts[k + 1], top if k > 0 else 0, bot if k < G - 1 else 0))
    for s in out:
        if s.hi - s.lo < top and G > 1:
            raise ValueError(f"strip {s.rank} owns {s.hi - s.lo} rows, fewer than the {top}-row "
                             f"halo its neighbour needs: use fewer ranks or a shorter segment")
    return out


def _weighted_cuts(w, G, min_rows):
    """Cut points 0 = c0 < c1 < ... < cG = H: cut k at the first row where the cumulative
    weight reaches k/G of the total, clamped so that every strip keeps >= min_rows rows."""
    H = len(w)
    if H < G * min_rows:
        raise ValueError(f"cannot split {H} rows into {G} strips of >= {min_rows} rows")
    if np.any(w < 0) or not np.all(np.isfinite(w)):
        raise ValueError("row weights must be finite and non-negative")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for k in range(1, G):
        c = int(np.searchsorted(cum, total * k / G, side="left")) if total > 0 else (H * k) // G
        lo = cuts[-1] + min_rows            # this strip keeps min_rows
        hi = H - (G - k) * min_rows         # the strips after it keep theirs
        cuts.append(min(max(c, lo), hi))
    cuts.append(H)
    return cuts


def row_weights(labels, floor: float = 1.0, cell=(8, 112)):
    """Per-row cost of a restricted solve from its band labels (2 = RD; `rds.Solver.labels()`
    after a K = 0 solve at the band's delta, or an oracle's).  cell = (rows, cols): the
    stencil's work unit, a band of `rows` rows by `cols` output columns, runs whole when it
    holds any RD pixel, so a row costs the active cells of its band, plus a
    floor for fixed per-row work.  cell = None: the row's RD pixel count (the compact path's
    cost)."""
    lab = np.asarray(labels) == 2
    if cell is None:
        return lab.sum(axis=1).astype(np.float64) + float(floor)
    ch, cw = int(cell[0]), int(cell[1])
    H, W = lab.shape
    nb, ns = -(-H // ch), -(-W // cw)
    pad = np.zeros((nb * ch, ns * cw), dtype=bool)
    pad[:H, :W] = lab
    active = pad.reshape(nb, ch, ns, cw).any(axis=(1, 3)).sum(axis=1).astype(np.float64)
    return np.repeat(active, ch)[:H] + float(floor)


def segments(iters: int, seg_iters: int) -> list[int]:
    """Iterations per segment: `seg_iters` each, the last one shorter."""
    full, rem = divmod(iters, seg_iters)
    return [seg_iters] * full + ([rem] if rem else [])


def exchange_plan(plan: list[Strip]) -> list[tuple[int, int, int, int, int]]:
    """Halo refresh as (src_rank, src_row, dst_rank, dst_row, nrows) copies in local row
    coordinates: every halo row comes from the rank that owns that global row."""
    out = []
    for k in range(len(plan) - 1):
        a, b = plan[k], plan[k + 1]  # a above b; a.hi == b.lo
        # b's top halo = a's last b.top owned rows
        out.append((a.rank, a.owned.stop - b.top, b.rank, 0, b.top))
        # a's bottom halo = b's first a.bot owned rows
        out.append((b.rank, b.top, a.rank, a.rows - a.bot, a.bot))
    return out


def solve_local(engines, plan, lam, theta, tau, delta, iters, seg_iters, device=None):
    """All strips in one process (one GPU, handles run one after another): the exchange
    copies the state rows through host buffers, or through torch tensors on `device`
    (stream-ordered, no synchronisation: the engines must then run on torch's current
    stream, so the caching allocator sees every use of a buffer).  Used to test and time the decomposition on a
    single device; `StripSolver` is the one-rank-per-GPU form."""
    xplan = exchange_plan(plan)
    for n, it in enumerate(segments(iters, seg_iters) or [0]):
        if n == 0:
            for e in engines:
                e.solve(lam, theta, tau, delta, it)
            continue
        if device is None:
            bufs = [(d, dr, engines[s].state_rows(sr, m)) for s, sr, d, dr, m in xplan]
        else:
            import torch

            bufs = []
            for s, sr, d, dr, m in xplan:
                W = engines[s].shape[1]
                buf = torch.empty((3, m, W), dtype=torch.float32, device=device)
                bufs.append((d, dr, engines[s].state_rows(sr, m, out=buf)))
        for d, dr, buf in bufs:
            engines[d].set_state_rows(dr, buf)
        for e in engines:
            e.solve_continue(it)


# ---- the paper's q -> q^ knob and stopping rule on a strip-decomposed image ----------------
# Both are global quantities (q^ is set by the fraction of ALL pixels;
# the norms run over the whole image), so every strip contributes its owned
# rows and the ranks combine them before a common decision.  The combination step is passed
# in (`allreduce`), so the same code runs over torch.distributed (StripSolver) and for several
# strip handles on one device (the *_local forms used by the tests).

def band_from_histograms(q, N, hist_pass):
    """q -> q^ as rds_band_for_fraction computes it: the smallest float32 q^ with
    #{|f| < q^} >= k = ceil(q N), i.e. the next float above the k-th smallest |f| (ties at the
    k-th value join RD).  `hist_pass(prefix, mask, shift)` returns the 256-bin histogram of
    byte `shift` of the |f| bit patterns matching `prefix` under `mask`, summed over the whole
    image; four passes from the top byte down find the k-th smallest bit pattern."""
    import math

    k = int(math.ceil(q * float(N)))
    k = min(k, N)
    if k <= 0:
        return np.float32(0.0)
    prefix, mask, rank = 0, 0, k
    for shift in (24, 16, 8, 0):
        hh = np.asarray(hist_pass(prefix, mask, shift), dtype=np.int64)
        c = np.cumsum(hh)
        d = int(np.searchsorted(c, rank))  # first bin whose cumulative count reaches rank
        if d >= 256:
            raise RuntimeError("histogram inconsistent")
        rank -= int(c[d - 1]) if d > 0 else 0
        prefix |= d << shift
        mask |= 255 << shift
    a = np.array([prefix], dtype=np.uint32).view(np.float32)[0]
    return np.nextafter(a, np.float32(np.inf), dtype=np.float32)


def tolerance_loop(run, allreduce, max_iters, tol, check_every, norm_div):
    """The stopping rule of PAPER.md:234-238 over strips: checks after iterations m, 2m, ...
    and at max_iters (m = check_every, reading R-F2), each on the all-reduced sums of the
    strips' owned rows.  `run(n, check)` advances every strip by n iterations (exchanging
    halos as it must) and, if check, returns this rank's (sum du^2, sum dv^2) of the last one.
    Returns dict(iters, residual, converged)."""
    import math

    done, r = 0, -1.0
    while done < max_iters:
        block = min(check_every, max_iters - done)
        su, sv = allreduce(run(block, True))
        done += block
        r = max(math.sqrt(su / norm_div), math.sqrt(sv / norm_div))
        if r <= tol:
            return dict(iters=done, residual=r, converged=1)
    return dict(iters=done, residual=r, converged=0)


def _chunks(n, seg_iters):
    """A block of n iterations as segments of at most seg_iters (a halo refresh before each
    but the first of the solve)."""
    out = []
    while n > 0:
        out.append(min(seg_iters, n))
        n -= out[-1]
    return out


def band_for_fraction_local(engines, plan, q, H, W):
    """q -> q^ of the whole image from strip handles on one device (histograms summed)."""
    def hist_pass(prefix, mask, shift):
        return sum(e.abs_histogram(st.owned.start, st.owned.stop, prefix, mask, shift)
                   .astype(np.int64) for st, e in zip(plan, engines))
    return band_from_histograms(q, H * W, hist_pass)


def solve_tol_local(engines, plan, lam, theta, tau, delta, max_iters, tol, check_every,
                    seg_iters, norm="l2"):
    """The tolerance solve of a strip-decomposed image with all strips in one process
    (exchange through host buffers, sums added in rank order)."""
    xplan = exchange_plan(plan)
    state = {"started": False}

    def exchange():
        bufs = [(d, dr, engines[s].state_rows(sr, m)) for s, sr, d, dr, m in xplan]
        for d, dr, buf in bufs:
            engines[d].set_state_rows(dr, buf)

    def run(n, check):
        chunks = _chunks(n, seg_iters)
        sums = None
        for k, it in enumerate(chunks):
            sums = _advance(engines, plan, state, exchange, lam, theta, tau, delta, it,
                            check and k == len(chunks) - 1)
        return sums

    def allreduce(parts):
        return tuple(float(sum(p[i] for p in parts)) for i in range(2))

    H = sum(st.hi - st.lo for st in plan)
    W = engines[0].shape[1]
    return tolerance_loop(run, allreduce, max_iters, tol, check_every,
                          float(H * W) if norm == "rms" else 1.0)


def _advance(engines, plan, state, exchange, lam, theta, tau, delta, it, check):
    """Advance this process's strips (`engines`, their `plan` entries) by `it` iterations: the
    solve's first segment sets up, later ones refresh the halos first.  With check, return
    every strip's owned-row sums (du^2, dv^2) of the last iteration."""
    if not state["started"]:
        for e in engines:
            e.solve(lam, theta, tau, delta, it - 1 if check else it)
        state["started"] = True
        if not check:
            return None
        it = 1  # the checked iteration continues the first segment (no refresh needed)
    else:
        exchange()
    if not check:
        for e in engines:
            e.solve_continue(it)
        return None
    return [e.continue_check(it, st.owned.start, st.owned.stop) for st, e in zip(plan, engines)]


class StripSolver:
    """This rank's strip of an H x W image, one process per GPU (torch.distributed
    initialised by the caller).  `engine` defaults to an `rds.Solver` on torch's current
    stream; tests pass a stand-in with the same methods."""

    def __init__(self, H, W, seg_iters, engine=None, group=None, weights=None, **solver_kw):
        import torch
        import torch.distributed as dist

        self.dist, self.torch, self.group = dist, torch, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.H, self.W, self.seg_iters = int(H), int(W), int(seg_iters)
        self.plan = partition(self.H, self.world, self.seg_iters, weights)
        self.me = self.plan[self.rank]
        self.xplan = exchange_plan(self.plan)
        nccl = dist.get_backend(group) == "nccl"
        self.device = torch.device("cuda", torch.cuda.current_device()) if nccl else \
            torch.device("cpu")
        if engine is None:
            from . import rds

            engine = rds.Solver(self.me.rows, self.W,
                                stream=torch.cuda.current_stream().cuda_stream, **solver_kw)
        self.engine = engine
        # exchange buffers in the engine's state precision (float32 for librds)
        self.dtype = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[
            np.dtype(getattr(engine, "state_dtype", np.float32))]

    # -- inputs: the full image or this strip's held rows ---------------------------------
    def _rows(self, a):
        if a is None:
            return None
        if a.shape[0] == self.H:
            a = a[self.me.r0: self.me.r0 + self.me.rows]
        if tuple(a.shape) != (self.me.rows, self.W):
            raise ValueError(f"expected ({self.H} or {self.me.rows}, {self.W}), got {a.shape}")
        return np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a.contiguous()

    def set_image(self, z):
        self.engine.set_image(self._rows(z))

    def set_fitting(self, c1, c2, gamma=0.0, P=None):
        self.engine.set_fitting(c1, c2, gamma, self._rows(P))

    def absmax(self):
        """Global max |f| (all-reduce max of the strips' exact float32 maxima)."""
        t = self.torch.tensor([float(self.engine.absmax())], dtype=self.torch.float64,
                              device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return np.float32(t.item())

    # -- the iteration ----------------------------------------------------------------------
    def _exchange(self):
        torch, dist = self.torch, self.dist
        ops, recvs = [], []
        for s, sr, d, dr, m in self.xplan:
            if s == self.rank:
                buf = torch.empty((3, m, self.W), dtype=self.dtype, device=self.device)
                self._get_rows(sr, m, buf)
                ops.append(dist.P2POp(dist.isend, buf, d, self.group))
            if d == self.rank:
                buf = torch.empty((3, m, self.W), dtype=self.dtype, device=self.device)
                ops.append(dist.P2POp(dist.irecv, buf, s, self.group))
                recvs.append((dr, buf))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for dr, buf in recvs:
            self.engine.set_state_rows(dr, buf if buf.is_cuda else buf.numpy())

    def _get_rows(self, r0, m, buf):
        if buf.is_cuda:
            self.engine.state_rows(r0, m, out=buf)
        else:
            buf.copy_(self.torch.from_numpy(self.engine.state_rows(r0, m)))

    def solve(self, lam, theta, tau, delta, iters):
        for n, it in enumerate(segments(int(iters), self.seg_iters) or [0]):
            if n == 0:
                self.engine.solve(lam, theta, tau, delta, it)
            else:
                self._exchange()
                self.engine.solve_continue(it)

    def band_for_fraction(self, q):
        """q -> q^ over the WHOLE image: each rank's radix-select histogram
        of its owned rows, all-reduced per pass -- the same q^ as rds_band_for_fraction on the
        whole image."""
        torch, dist = self.torch, self.dist

        def hist_pass(prefix, mask, shift):
            h = self.engine.abs_histogram(self.me.owned.start, self.me.owned.stop, prefix, mask,
                                          shift)
            t = torch.as_tensor(np.asarray(h, np.int64), device=self.device)
            dist.all_reduce(t, group=self.group)
            return t.cpu().numpy()

        return band_from_histograms(q, self.H * self.W, hist_pass)

    def solve_q(self, lam, theta, tau, q, iters):
        self.solve(lam, theta, tau, self.band_for_fraction(q), iters)

    def solve_tol(self, lam, theta, tau, delta, max_iters, tol, check_every, norm="l2"):
        """The paper's stopping rule on the strip-decomposed image: checks
        after every check_every iterations and at max_iters, each deciding on the all-reduced
        owned-row sums, so every rank stops at the same iteration as a whole-image solve
        (reading R-F2: Euclidean norm, or "rms").  Returns dict(iters, residual, converged)."""
        torch, dist = self.torch, self.dist
        state = {"started": False}

        def run(n, check):
            chunks = _chunks(n, self.seg_iters)
            sums = None
            for k, it in enumerate(chunks):
                sums = _advance([self.engine], [self.me], state, self._exchange, lam, theta,
                                tau, delta, it, check and k == len(chunks) - 1)
            return sums[0] if sums else None

        def allreduce(s):
            t = torch.tensor([float(s[0]), float(s[1])], dtype=torch.float64, device=self.device)
            dist.all_reduce(t, group=self.group)
            return tuple(t.tolist())

        return tolerance_loop(run, allreduce, int(max_iters), float(tol), int(check_every),
                              float(self.H * self.W) if norm == "rms" else 1.0)

    # -- outputs: owned rows ----------------------------------------------------------------
    def u(self):
        return self.engine.u()[self.me.owned]

    def mask(self):
        return self.engine.mask()[self.me.owned]

    def energy(self):
        """Whole-image energies: the strips' owned-row sums of TV(v), lambda<f, v>, E(u) and
        D(rho), all-reduced (the gap and E(v) recomputed from the sums)."""
        self.engine.set_energy_rows(self.me.owned.start, self.me.owned.stop)
        e = self.engine.energy()
        keys = ("TV_v", "fit_v", "E_u", "D_p", "F_rd")
        t = self.torch.tensor([e.get(k, 0.0) for k in keys], dtype=self.torch.float64,
                              device=self.device)
        self.dist.all_reduce(t, group=self.group)
        tv, fit, eu, dp, frd = t.tolist()
        return dict(E_v=tv + fit, E_u=eu, D_p=dp, gap=tv + fit - dp, TV_v=tv, fit_v=fit,
                    F_rd=frd)

    def gather_u(self, dst=0):
        """The whole u on rank `dst` (None elsewhere); strips padded to the tallest."""
        torch, dist = self.torch, self.dist
        sizes = [s.hi - s.lo for s in self.plan]
        u = np.asarray(self.u())
        mine = torch.zeros((max(sizes), self.W), dtype=torch.float64, device=self.device)
        mine[: u.shape[0]] = torch.from_numpy(u.astype(np.float64)).to(self.device)
        if self.rank == dst:
            parts = [torch.empty_like(mine) for _ in sizes]
            dist.gather(mine, parts, dst=dst, group=self.group)
            return np.concatenate([p[:n].cpu().numpy() for p, n in zip(parts, sizes)])
        dist.gather(mine, None, dst=dst, group=self.group)
        return None
