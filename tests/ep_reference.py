"""Test-only reference of the expert-parallel placement and exchange tables
(include/brownout.h "Expert parallelism"), written in plain
Python/numpy from the placement rule and the layouts the header documents.
The library computes the same on the host (placement, bo_ep_placement) and on
the device (tables, k_ep_tables); the tests compare both against this.

Placement: original expert e on rank floor(e R / m); united expert j (group j =
experts [j*way, min((j+1)*way, m))) f-sliced over the distinct owner
ranks of its members when every group has the same number n of them and f / n
is a multiple of 128, else whole on the owner of its first member.  Virtual
executors are rank-major: per rank its originals ascending, then its slices.
"""
from __future__ import annotations

import numpy as np


class EPPlanner:
    def __init__(self, m: int, way: int, f: int, world: int, align: int = 128):
        self.m, self.way, self.f, self.R = m, way, f, world
        self.G = -(-m // way)
        self.owner = [(e * world) // m for e in range(m)]
        gowners = [sorted({self.owner[e] for e in range(j * way, min((j + 1) * way, m))}) for j in range(self.G)]
        ns = {len(o) for o in gowners}
        self.sliced = len(ns) == 1 and all(f % (n * align) == 0 for n in ns)
        if not self.sliced:
            gowners = [[self.owner[j * way]] for j in range(self.G)]
        self.group_owners = gowners
        self.n_slices = len(gowners[0])
        self.f_u = f // self.n_slices
        self.nrep = self.n_slices
        self.vexec = []          # (rank, kind, idx, slice)
        for q in range(world):
            for e in range(m):
                if self.owner[e] == q:
                    self.vexec.append((q, "o", e, 0))
            for j in range(self.G):
                if q in gowners[j]:
                    self.vexec.append((q, "u", j, gowners[j].index(q)))
        self.V = len(self.vexec)
        self.v_of_orig = {e: v for v, (q, k, e, s) in enumerate(self.vexec) if k == "o"}
        self.v_of_slice = {(j, s): v for v, (q, k, j, s) in enumerate(self.vexec) if k == "u"}
        self.local_v = [[v for v, t in enumerate(self.vexec) if t[0] == q] for q in range(world)]

    def local_experts(self, q: int):
        es = [e for e in range(self.m) if self.owner[e] == q]
        return (es[0], es[-1] + 1) if es else (0, 0)

    def local_slices(self, q: int):
        return [(self.vexec[v][2], self.vexec[v][3]) for v in self.local_v[q] if self.vexec[v][1] == "u"]

    def feeds(self, exec_of_expert):
        """Experts (ascending) whose rows each virtual executor processes under the plan."""
        fd = [[] for _ in range(self.V)]
        for e in range(self.m):
            x = int(exec_of_expert[e])
            if x < 0:
                continue
            if x < self.m:
                fd[self.v_of_orig[x]].append(e)
            else:
                j = x - self.m
                for s in range(len(self.group_owners[j])):
                    fd[self.v_of_slice[(j, s)]].append(e)
        return fd

    def tables(self, C, exec_of_expert, q, padded=False, cap=0):
        """Exchange tables of rank q for gathered counts C [R, m] and the global
        plan's executor map, in the layouts of include/brownout.h."""
        C = np.asarray(C, dtype=np.int64)
        R, m, V = self.R, self.m, self.V
        fd = self.feeds(exec_of_expert)
        rows = np.zeros((R, V), dtype=np.int64)
        for v in range(V):
            for e in fd[v]:
                rows[:, v] += C[:, e]
        vrank = np.array([t[0] for t in self.vexec])
        # source side (q sends): segment of each v in q's send buffer
        base = np.zeros(V, dtype=np.int64)
        for d in range(R):
            off = d * cap if padded else int(rows[q, vrank < d].sum())
            for v in np.nonzero(vrank == d)[0]:
                base[v] = off
                off += rows[q, v]
        send = np.array([rows[q, vrank == d].sum() for d in range(R)], dtype=np.int64)
        row_base = np.full((m, self.nrep), -1, dtype=np.int64)
        for v in range(V):
            acc = 0
            for e in fd[v]:
                x = int(exec_of_expert[e])
                rep = 0 if x < m else self.vexec[v][3]
                row_base[e, rep] = base[v] + acc
                acc += C[q, e]
        # destination side (q receives)
        lv = self.local_v[q]
        nl = len(lv)
        recv = np.array([rows[r, lv].sum() for r in range(R)], dtype=np.int64)
        rbase = [r * cap if padded else int(recv[:r].sum()) for r in range(R)]
        recv_blk = np.zeros((R, nl), dtype=np.int64)
        for r in range(R):
            off = rbase[r]
            for i, v in enumerate(lv):
                recv_blk[r, i] = off
                off += rows[r, v]
        grp_blk = np.zeros((nl, R), dtype=np.int64)
        off = 0
        exec_off = [0]
        for i, v in enumerate(lv):
            for r in range(R):
                grp_blk[i, r] = off
                off += rows[r, v]
            exec_off.append(off)
        exec_off = np.array(exec_off, dtype=np.int64)
        ex_rows = np.diff(exec_off)
        mtile_off = np.concatenate([[0], np.cumsum((ex_rows + 127) // 128)])
        length = np.array([[rows[r, v] for v in lv] for r in range(R)], dtype=np.int64).reshape(R, nl)
        extent = R * cap if padded else int(recv.sum())
        return dict(
            row_base=row_base.reshape(-1), send_rows=send, recv_rows=recv,
            fwd_dst=np.append(grp_blk.reshape(-1), off), fwd_len=length.T.reshape(-1), fwd_src=recv_blk.T.reshape(-1),
            inv_dst=np.append(recv_blk.reshape(-1), extent), inv_len=length.reshape(-1), inv_src=grp_blk.T.reshape(-1),
            exec_off=exec_off, mtile_off=mtile_off, totals=np.array([off, extent], dtype=np.int64),
            n_orig=sum(1 for v in lv if self.vexec[v][1] == "o"), n_united=sum(1 for v in lv if self.vexec[v][1] == "u"),
            rows=rows)


TABLE_ORDER = ("row_base", "send_rows", "recv_rows", "fwd_dst", "fwd_len", "fwd_src", "inv_dst", "inv_len", "inv_src",
               "exec_off", "mtile_off", "totals")


def split_tables(flat, m, nrep, R, nl):
    """Cut the device int32 table block (include/brownout.h order) into named arrays."""
    nb = nl * R
    sizes = dict(row_base=m * nrep, send_rows=R, recv_rows=R, fwd_dst=nb + 1, fwd_len=nb, fwd_src=nb, inv_dst=nb + 1,
                 inv_len=nb, inv_src=nb, exec_off=nl + 1, mtile_off=nl + 1, totals=2)
    out, o = {}, 0
    for k in TABLE_ORDER:
        out[k] = np.asarray(flat[o:o + sizes[k]])
        o += sizes[k]
    return out
