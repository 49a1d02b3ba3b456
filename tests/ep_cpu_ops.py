"""Test-only CPU stand-in for paper_2507_17133_b200.ep.EPContext.

Implements the stage calls of the library's EP API (route, dispatch, splits,
compute, combine and the workspace views the exchanges read and write) with
plain torch / numpy on the CPU, so that the expert-parallel orchestration
(ep.ep_forward_staged: count all-gather, exact / padded split sizes, dispatch
and return all-to-all, f-slice partial sums) runs with gloo process groups on
a machine without a GPU.  Routing and Alg. 1 come from the oracle and the
tables from tests/ep_reference.py; nothing here is on the product path.
"""
import struct

import numpy as np
import torch

from oracle import brownout_oracle as O
from tests.ep_reference import EPPlanner


class CpuEPContext:
    def __init__(self, m, f, d, K, way, world, rank, max_tokens, ratio, mode=O.PARTIAL, padded=False,
                 dtype=torch.float32):
        self.m, self.f, self.d, self.K, self.way = m, f, d, K, way
        self.world, self.rank = world, rank
        self.ratio, self.mode = ratio, mode
        self.pl = EPPlanner(m, way, f, world)
        self.cap = max_tokens * K
        self.padded = padded
        self.rows_max = world * self.cap
        self.dtype = dtype
        self._row = torch.zeros(m + 4, dtype=torch.int32)
        self._gathered = torch.zeros(world * (m + 4), dtype=torch.int32)
        self.send = torch.zeros(self.rows_max, d, dtype=dtype)
        self.send_w = torch.zeros(self.rows_max, dtype=torch.float32)
        self.recv = torch.zeros(self.rows_max, d, dtype=dtype)
        self.recv_w = torch.zeros(self.rows_max, dtype=torch.float32)
        self.slices = self.pl.local_slices(rank)

    def local_weights(self, experts, united):
        Wg, Wu, Wd = experts
        e0, e1 = self.pl.local_experts(self.rank)
        ex = (Wg[e0:e1], Wu[e0:e1], Wd[e0:e1]) if e1 > e0 else None
        if not self.slices:
            return ex, None
        UWg, UWu, UWd = united
        fu = self.pl.f_u
        return ex, (torch.stack([UWg[j, s * fu:(s + 1) * fu, :] for j, s in self.slices]),
                    torch.stack([UWu[j, s * fu:(s + 1) * fu, :] for j, s in self.slices]),
                    torch.stack([UWd[j, :, s * fu:(s + 1) * fu] for j, s in self.slices]))

    def count_row(self):
        return self._row

    def gathered(self):
        return self._gathered

    def rows(self, name):
        return self.send if name == "send" else self.recv

    def weights(self, name):
        return self.send_w if name == "send" else self.recv_w

    def route(self, x, Wr, logits=None):
        L = np.asarray(logits, dtype=np.float64) if logits is not None else O.router_logits(
            x.double().numpy(), Wr.double().numpy())
        self.T = x.shape[0]
        self.ids, self.g = O.topk_gate(L, self.K)
        cnt = O.expert_counts(self.ids, self.m)
        lo, hi = struct.unpack("<ii", struct.pack("<d", self.ratio))
        self._row[:] = torch.as_tensor(list(cnt) + [self.T, 1 if self.mode == O.FULL else 0, lo, hi],
                                       dtype=torch.int32)
        return self._row

    def dispatch(self, x):
        G = self._gathered.view(self.world, self.m + 4).numpy()
        C = G[:, :self.m]
        lo, hi = int(G[0, self.m + 2]), int(G[0, self.m + 3])   # rank 0's knob (D18 + the EP contract)
        ratio = struct.unpack("<d", struct.pack("<ii", lo, hi))[0]
        mode = O.FULL if G[0, self.m + 1] else O.PARTIAL
        self.plan = O.brownout_plan(C.sum(0), ratio, self.way, mode)
        self.tab = self.pl.tables(C, self.plan.exec_of_expert, self.rank, self.padded, self.cap)
        rb = self.tab["row_base"].reshape(self.m, self.pl.nrep)
        nxt = np.zeros(self.m, dtype=np.int64)
        self.row_of = np.full(self.T * self.K * self.pl.nrep, -1, dtype=np.int64)
        for t in range(self.T):
            for s in range(self.K):
                e = int(self.ids[t, s])
                rank = nxt[e]
                nxt[e] += 1
                for rep in range(self.pl.nrep):
                    if rb[e, rep] >= 0:
                        r = int(rb[e, rep] + rank)
                        self.send[r] = x[t]
                        self.send_w[r] = float(self.g[t, s])
                        self.row_of[(t * self.K + s) * self.pl.nrep + rep] = r

    def splits(self):
        if self.padded:
            return [self.cap] * self.world, [self.cap] * self.world
        return [int(v) for v in self.tab["send_rows"]], [int(v) for v in self.tab["recv_rows"]]

    def _blocks(self, src, dst, dst_start, length, src_off, w_src=None, w_dst=None):
        for b in range(len(length)):
            n = int(length[b])
            if n:
                d0, s0 = int(dst_start[b]), int(src_off[b])
                dst[d0:d0 + n] = src[s0:s0 + n]
                if w_src is not None:
                    w_dst[d0:d0 + n] = w_src[s0:s0 + n]

    def compute(self, local_experts, local_united):
        tb = self.tab
        grouped = torch.zeros(self.rows_max, self.d, dtype=self.dtype)
        gw = torch.zeros(self.rows_max, dtype=torch.float32)
        self._blocks(self.recv, grouped, tb["fwd_dst"], tb["fwd_len"], tb["fwd_src"], self.recv_w, gw)
        eo = tb["exec_off"]
        n_o = tb["n_orig"]
        out = torch.zeros_like(grouped)
        for i in range(len(eo) - 1):
            r0, r1 = int(eo[i]), int(eo[i + 1])
            if r1 == r0:
                continue
            Wg, Wu, Wd = (w[i] for w in local_experts) if i < n_o else (w[i - n_o] for w in local_united)
            X = grouped[r0:r1].double()
            h = torch.nn.functional.silu(X @ Wg.double().T) * (X @ Wu.double().T)
            out[r0:r1] = (gw[r0:r1].double()[:, None] * (h @ Wd.double().T)).to(out.dtype)
        self._blocks(out, self.recv, tb["inv_dst"], tb["inv_len"], tb["inv_src"])   # ret aliases recv

    def combine(self, x):
        y = torch.zeros_like(x)
        ro = self.row_of.reshape(self.T, -1)
        for t in range(self.T):
            acc = torch.zeros(self.d, dtype=torch.float64)
            for r in ro[t].tolist():
                if r >= 0:
                    acc += self.send[r].double()   # back aliases send
            y[t] = acc.to(y.dtype)
        return y
