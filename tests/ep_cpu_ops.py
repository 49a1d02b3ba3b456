"""Test-only CPU backend for paper_2507_17133_b200.ep.EPMoE.

Implements the seven building-block calls of the C ABI (route, local_counts,
plan_counts, dispatch, block_copy, expert_ffn, combine) with plain torch /
numpy on the CPU so that the expert-parallel orchestration (placement, count
all-gather, split sizes, dispatch / combine all-to-all, regrouping, f-slice
partial sums) can be exercised with gloo process groups on a machine with no
GPU.  Routing and Alg. 1 come from the oracle (tests may use it); nothing here
is on the product path.
"""
import numpy as np
import torch

from oracle import brownout_oracle as O


class CpuOps:
    def __init__(self, m, K, way, ratio, mode=O.PARTIAL):
        self.m, self.K, self.way, self.ratio, self.mode = m, K, way, ratio, mode

    def route(self, x, Wr, logits=None):
        L = np.asarray(logits, dtype=np.float64) if logits is not None else O.router_logits(
            x.double().numpy(), Wr.double().numpy())
        ids, g = O.topk_gate(L, self.K)
        return {"ids": ids, "g": g, "counts": O.expert_counts(ids, self.m)}

    def local_counts(self, T, ws):
        return torch.as_tensor(ws["counts"], dtype=torch.int32)

    def plan_counts(self, C):
        tot = C.to(torch.int64).sum(0).numpy()
        p = O.brownout_plan(tot, self.ratio, self.way, self.mode)
        return {"exec_of_expert": torch.as_tensor(p.exec_of_expert, dtype=torch.int32)}

    def dispatch(self, T, row_base, nrep, x, rows_out, w_out, row_of, workspace=None):
        ws = workspace
        rb = row_base.numpy().reshape(self.m, nrep)
        nxt = np.zeros(self.m, dtype=np.int64)
        row_of.fill_(-1)
        for t in range(T):
            for s in range(self.K):
                e = int(ws["ids"][t, s])
                rank = nxt[e]
                nxt[e] += 1
                for rep in range(nrep):
                    if rb[e, rep] >= 0:
                        r = int(rb[e, rep] + rank)
                        rows_out[r] = x[t]
                        w_out[r] = float(ws["g"][t, s])
                        row_of[(t * self.K + s) * nrep + rep] = r

    def block_copy(self, src, dst, src_off, dst_start, w_src=None, w_dst=None):
        so, ds = src_off.tolist(), dst_start.tolist()
        for b in range(len(so)):
            n = ds[b + 1] - ds[b]
            if n:
                dst[ds[b]:ds[b] + n] = src[so[b]:so[b] + n]
                if w_src is not None:
                    w_dst[ds[b]:ds[b] + n] = w_src[so[b]:so[b] + n]

    def expert_ffn(self, rows, row_w, exec_off, mtile_off, n_orig, n_united, f_united, experts, united, h_buf, out):
        eo = exec_off.tolist()
        for i in range(n_orig + n_united):
            r0, r1 = eo[i], eo[i + 1]
            if r1 == r0:
                continue
            Wg, Wu, Wd = (w[i] for w in experts) if i < n_orig else (w[i - n_orig] for w in united)
            X = rows[r0:r1].double()
            h = torch.nn.functional.silu(X @ Wg.double().T) * (X @ Wu.double().T)
            out[r0:r1] = (row_w[r0:r1].double()[:, None] * (h @ Wd.double().T)).to(out.dtype)

    def combine(self, T, rows, row_of, nrep, x, y):
        ro = row_of.view(T, -1)
        for t in range(T):
            acc = torch.zeros(rows.shape[1], dtype=torch.float64)
            for r in ro[t].tolist():
                if r >= 0:
                    acc += rows[r].double()
            y[t] = acc.to(y.dtype)
