"""CPU stand-in for paper_2502_02704_b200.parareal.GpuBackend (TESTS ONLY).

Same interface (empty / jumps / correct / nx / times / device), arithmetic from
the oracle, so the rank decomposition and the jump exchange of ShardedRun can
be exercised with the gloo backend on a CPU-only host.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import bgk as O


def key(unit, step, kind):
    return (unit << 40) | (step << 8) | kind


def pack(U):
    rho, u, th = U
    out = np.empty((5, rho.shape[0]))
    out[0], out[1:4], out[4] = rho, np.asarray(u).T, th
    return torch.from_numpy(out)


def unpack(t):
    m = t.numpy()
    return m[0].copy(), np.ascontiguousarray(m[1:4].T), m[4].copy()


class OracleBackend:
    def __init__(self, prob: O.Problem, fail_window: int | None = None):
        self.prob = prob
        self.nx = prob.mesh.nx
        self.times = [float(t) for t in prob.times]
        self.device = torch.device("cpu")
        self.fail_window = fail_window
        self.t_kin = self.t_fluid = 0.0
        self.windows_done = []

    def empty(self, n):
        return torch.empty((n, 5, self.nx), dtype=torch.float64)

    def jumps(self, snaps, windows, out):
        codes = []
        for w, n in enumerate(windows):
            self.windows_done.append(n)
            if n == self.fail_window:
                codes.append(key(0, 2, 2))  # BlowUpError(step=2)
                continue
            out[w] = pack(O.window_jump(self.prob, unpack(snaps[n - 1]), n))
            codes.append(-1)
        return codes

    def correct(self, snaps, old, jumps, start):
        err = 0.0
        for n in range(start, len(self.times)):
            cor = O._add(O.G(self.prob, unpack(snaps[n - 1]), n), unpack(jumps[n - 1]))
            ok = all(np.all(np.isfinite(x)) for x in cor)
            if not ok or np.any(cor[0] <= 0.0) or np.any(cor[2] <= 0.0):
                return 0.0, key(n, 0, 4)
            err = max(err, O.sup_gap(cor, unpack(old[n])))
            snaps[n] = pack(cor)
        return err, -1

    # -- pipelined interface (PipelinedRun), synchronous on the CPU ----------
    def fine_into(self, src, n, out):
        self.windows_done.append(n)
        if n == self.fail_window:
            out.fill_(float("nan"))
            return key(0, 2, 2)  # BlowUpError(step=2)
        out.copy_(pack(O.PFL(self.prob, unpack(src), n)))
        return -1

    def side_begin(self, snaps):
        self._gst = [-1] * (len(self.times) - 1)
        self._cst = -1
        self._emax = 0.0
        return snaps.clone()

    def round_slot(self, r, nslots):
        return torch.empty((nslots, 5, self.nx), dtype=torch.float64)

    def side_round(self, r, fine, windows, snaps, old, jumps):
        for q, n in enumerate(windows):
            try:
                G = O.G(self.prob, unpack(old[n - 1]), n)
            except O.OracleError:
                self._gst[n - 1] = key(0, 1, 2)
                continue
            jumps[n - 1] = pack(O._sub(unpack(fine[q]), G))
        for n in windows:
            if self._cst >= 0:
                return
            try:
                Gn = O.G(self.prob, unpack(snaps[n - 1]), n)
            except O.OracleError:
                self._cst = key(n, 1, 3)
                return
            cor = O._add(Gn, unpack(jumps[n - 1]))
            ok = all(np.all(np.isfinite(x)) for x in cor)
            if not ok or np.any(cor[0] <= 0.0) or np.any(cor[2] <= 0.0):
                self._cst = key(n, 0, 4)
                return
            self._emax = max(self._emax, O.sup_gap(cor, unpack(old[n])))
            snaps[n] = pack(cor)

    def side_finish(self):
        return self._emax, list(self._gst), self._cst
