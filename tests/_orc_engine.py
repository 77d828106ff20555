"""Test stand-in for an rds.Solver strip handle, backed by the CPU oracle (fp64 state): the
methods `paper_1807_11534_b200.strips` calls, so the strip protocol can be checked on CPU
against a whole-image oracle solve."""
import numpy as np

import oracle


class OracleEngine:
    state_dtype = np.float64

    def __init__(self, H, W):
        self.shape = (H, W)
        self.f = None
        self.z = None
        self.st = None
        self.e_rows = (0, H)

    def set_image(self, z):
        self.z = np.asarray(z, np.float32)

    def set_fitting(self, c1, c2, gamma=0.0, P=None):
        self.f = oracle.fitting(self.z, c1, c2, gamma, P)

    def absmax(self):
        return oracle.absmax(self.f)

    def solve(self, lam, theta, tau, delta, iters):
        self.par = (delta, lam, theta, tau)
        self.st = oracle.solve(self.f, delta, lam, theta, tau, iters)

    def solve_continue(self, iters):
        delta, lam, theta, tau = self.par
        s = self.st
        self.st = oracle.solve(self.f, delta, lam, theta, tau, iters,
                               init=(s["v"], s["p1"], s["p2"]))

    def state_rows(self, r0, n, out=None):
        s = self.st
        return np.stack([s["v"][r0:r0 + n], s["p1"][r0:r0 + n], s["p2"][r0:r0 + n]])

    def set_state_rows(self, r0, buf):
        buf = np.asarray(buf, np.float64)
        for k, name in enumerate(("v", "p1", "p2")):
            self.st[name][r0:r0 + buf.shape[1]] = buf[k]

    def continue_check(self, iters, r0, r1):
        """rds_continue_check: `iters` more iterations, then the stopping-rule sums of the
        last one over rows [r0, r1)."""
        if iters > 1:
            self.solve_continue(iters - 1)
        up, vp = self.st["u"].copy(), self.st["v"].copy()
        self.solve_continue(1)
        du = self.st["u"][r0:r1] - up[r0:r1]
        dv = self.st["v"][r0:r1] - vp[r0:r1]
        return float(np.sum(du * du)), float(np.sum(dv * dv))

    def abs_histogram(self, r0, r1, prefix, mask, shift):
        """rds_abs_histogram: byte `shift` of the |f| bit patterns of rows [r0, r1) matching
        prefix under mask."""
        b = np.abs(self.f[r0:r1]).view(np.uint32).ravel()
        b = b[(b & np.uint32(mask)) == np.uint32(prefix)]
        return np.bincount((b >> np.uint32(shift)) & np.uint32(255), minlength=256).astype(
            np.int64)

    def u(self):
        return self.st["u"]

    def mask(self):
        return (self.st["u"] > 0.5).astype(np.uint8)
