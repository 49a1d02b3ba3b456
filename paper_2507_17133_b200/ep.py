"""Expert-parallel (EP) brownout MoE forward over R ranks.

One process per GPU.  Tokens are data-parallel (each rank owns a contiguous
slice of the global batch); experts are sharded:

  * original expert e lives on rank owner(e) = floor(e * R / m);
  * united expert j (group j = experts [j*way, min((j+1)*way, m))) is
    f-sliced across the distinct owner ranks of its members, so that a ratio-1
    step (every row on united experts) still keeps every rank busy.  SwiGLU is
    elementwise in f, so the slices' partial outputs simply add in the combine.
    When the groups' owner counts differ (or f/n is not a multiple of 128) the
    united expert lives whole on the owner of its first member instead.

The plan is global (reading D18): every rank all-gathers the per-rank expert
counts, and Alg. 1 runs on their sum, so EP over R ranks computes exactly the
single-GPU forward of the rank-order concatenated batch.

Data path per forward on rank r (kernels are the C-ABI building blocks; the
exchanges are torch.distributed collectives — NCCL over NVLink on the B200 box,
gloo in the CPU tests):

  1. bo_route          router + top-K + local counts                (kernels)
  2. all_gather        counts [R, m]                                 (NCCL)
  3. bo_plan_counts    Alg. 1 on the global counts                   (kernel)
     D2H of counts + executor map (one host sync), host tables (below)
  4. bo_dispatch       rows ordered (virtual executor, expert, token) = per-destination segments
  5. all_to_all        rows + gate weights to their executor ranks   (NCCL)
  6. bo_block_copy     (source, executor) -> (executor, source) order
  7. bo_expert_ffn     grouped SwiGLU GEMMs (tcgen05) on local executors
  8. bo_block_copy     back to (source, executor) order
  9. all_to_all        weighted outputs back to the token owners     (NCCL)
 10. bo_combine        y_t = sum over slots and slices               (kernel)

Everything here is host-side bookkeeping (numpy on tiny [R, m] tables) and
argument marshalling; no step of the method's arithmetic runs in Python.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


class EPPlanner:
    """Static expert placement and the per-forward exchange tables (host logic)."""

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
        self.n_slices = len(gowners[0]) if self.sliced else 1
        self.f_u = f // self.n_slices
        self.nrep = max(len(o) for o in gowners)
        # virtual executors, rank-major: per rank its originals (ascending), then its united slices
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

    # -- static local weights ------------------------------------------------
    def local_experts(self, q: int):
        es = [e for e in range(self.m) if self.owner[e] == q]
        return (es[0], es[-1] + 1) if es else (0, 0)

    def local_slices(self, q: int):
        return [(self.vexec[v][2], self.vexec[v][3]) for v in self.local_v[q] if self.vexec[v][1] == "u"]

    def local_weights(self, q: int, experts, united):
        """Views / copies of the weights rank q executes: originals [e0, e1) and
        the f-slices of its united experts, stacked."""
        Wg, Wu, Wd = experts
        e0, e1 = self.local_experts(q)
        ex = (Wg[e0:e1], Wu[e0:e1], Wd[e0:e1])
        sl = self.local_slices(q)
        if not sl or united is None:
            return ex, None
        UWg, UWu, UWd = united
        fu = self.f_u
        ug = torch.stack([UWg[j, s * fu:(s + 1) * fu, :] for j, s in sl]).contiguous()
        uu = torch.stack([UWu[j, s * fu:(s + 1) * fu, :] for j, s in sl]).contiguous()
        ud = torch.stack([UWd[j, :, s * fu:(s + 1) * fu] for j, s in sl]).contiguous()
        return ex, (ug, uu, ud)

    # -- per-forward tables -----------------------------------------------------
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

    def tables(self, C, exec_of_expert, rank=None):
        """C [R, m] per-rank expert counts; exec_of_expert [m] of the global plan.
        Returns the per-rank tables of every rank, or only rank `rank`'s (the
        forward path: each rank builds just its own)."""
        C = np.asarray(C, dtype=np.int64)
        R, m, V = self.R, self.m, self.V
        fd = self.feeds(exec_of_expert)
        rows = np.zeros((R, V), dtype=np.int64)          # rows[r][v]
        for v in range(V):
            for e in fd[v]:
                rows[:, v] += C[:, e]
        vstart = np.zeros((R, V), dtype=np.int64)        # send-buffer start of v on source r
        vstart[:, 1:] = np.cumsum(rows, axis=1)[:, :-1]
        vrank = np.array([t[0] for t in self.vexec])
        send = np.zeros((R, R), dtype=np.int64)          # send[r][q]
        for q in range(R):
            send[:, q] = rows[:, vrank == q].sum(axis=1)
        # row_base[r][e][rep]
        row_base = np.full((R, m, self.nrep), -1, dtype=np.int64)
        for v in range(V):
            acc = np.zeros(R, dtype=np.int64)
            for e in fd[v]:
                x = int(exec_of_expert[e])
                rep = 0 if x < m else self.vexec[v][3]
                row_base[:, e, rep] = vstart[:, v] + acc
                acc += C[:, e]
        per_rank = []
        for q in (range(R) if rank is None else (rank,)):
            lv = self.local_v[q]
            # receive buffer: source-major, then local executor order
            recv_seg = np.concatenate([[0], np.cumsum(send[:, q])])
            recv_blk = np.zeros((R, len(lv)), dtype=np.int64)
            for r in range(R):
                off = recv_seg[r]
                for i, v in enumerate(lv):
                    recv_blk[r, i] = off
                    off += rows[r, v]
            # grouped buffer: local executor major, then source
            grp_blk = np.zeros((len(lv), R), dtype=np.int64)
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
            # regroup: dst = grouped order (v, r), src = recv offsets
            fwd_dst_start = np.append(grp_blk.reshape(-1), off)
            fwd_src_off = recv_blk.T.reshape(-1)                 # (v, r) order
            # inverse: dst = recv order (r, v), src = grouped offsets
            inv_dst_start = np.append(recv_blk.reshape(-1), recv_seg[-1])
            inv_src_off = grp_blk.T.reshape(-1)                  # (r, v) order
            n_orig = sum(1 for v in lv if self.vexec[v][1] == "o")
            per_rank.append(dict(
                row_base=row_base[q].reshape(-1), send_splits=send[q].tolist(), recv_splits=send[:, q].tolist(),
                R_send=int(send[q].sum()), R_recv=int(send[:, q].sum()),
                fwd_src_off=fwd_src_off, fwd_dst_start=fwd_dst_start,
                inv_src_off=inv_src_off, inv_dst_start=inv_dst_start,
                exec_off=exec_off, mtile_off=mtile_off, n_orig=n_orig, n_united=len(lv) - n_orig))
        return per_rank if rank is None else per_rank[0]


class TorchComm:
    """Exchange over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo cannot move CUDA tensors: stage through host memory (test rigs only)
        self.stage = dist.get_backend(group) == "gloo"

    def _host(self, t):
        return t.cpu() if (self.stage and t.is_cuda) else t

    def all_gather_counts(self, local: torch.Tensor) -> torch.Tensor:
        src = self._host(local.contiguous())
        out = torch.empty(self.world * local.numel(), dtype=local.dtype, device=src.device)
        self.dist.all_gather_into_tensor(out, src, group=self.group)
        return out.view(self.world, -1).to(local.device)

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        o = self._host(out)
        self.dist.all_to_all_single(o, self._host(inp), output_split_sizes=list(out_splits),
                                    input_split_sizes=list(in_splits), group=self.group)
        if o is not out:
            out.copy_(o)


@dataclass
class EPState:
    T: int
    tabs: dict
    row_of: torch.Tensor
    send_x: torch.Tensor
    send_w: torch.Tensor


class EPMoE:
    """Expert-parallel brownout MoE layer on one rank.

    ``ops`` is the compute backend: a BrownoutMoE handle (the C-ABI CUDA path)
    in production; tests may pass a CPU implementation of the same six calls
    (route / local_counts / plan_counts / dispatch / block_copy / expert_ffn /
    combine) to exercise this orchestration with gloo."""

    TABLE_KEYS = ("row_base", "fwd_src_off", "fwd_dst_start", "inv_src_off", "inv_dst_start", "exec_off",
                  "mtile_off")

    def __init__(self, ops, planner: EPPlanner, rank: int, experts, united, d: int, K: int, dtype):
        self.ops, self.pl, self.rank = ops, planner, rank
        self.d, self.K, self.dtype = d, K, dtype
        self.ex, self.un = planner.local_weights(rank, experts, united)
        self._h_tab = None   # persistent (pinned on GPUs) host staging of the per-forward int32 tables
        self._d_tab = None

    def _upload_tables(self, tabs, dev):
        """All int32 tables of this forward in ONE host-to-device copy (one staging
        buffer reused every forward; the D2H of the next forward's counts orders it)."""
        parts = [np.asarray(tabs[k], dtype=np.int32).reshape(-1) for k in self.TABLE_KEYS]
        n = sum(a.size for a in parts)
        if self._h_tab is None or self._h_tab.numel() < n:
            cap = max(n, 1024) * 2
            self._h_tab = torch.empty(cap, dtype=torch.int32)
            if dev.type == "cuda":
                self._h_tab = self._h_tab.pin_memory()
            self._d_tab = torch.empty(cap, dtype=torch.int32, device=dev)
        hv = self._h_tab.numpy()
        views, o = {}, 0
        for k, a in zip(self.TABLE_KEYS, parts):
            hv[o:o + a.size] = a
            views[k] = (o, a.size)
            o += a.size
        self._d_tab[:n].copy_(self._h_tab[:n], non_blocking=True)
        return {k: self._d_tab[o0:o0 + sz] for k, (o0, sz) in views.items()}

    # phase 1 --------------------------------------------------------------
    def route(self, x, Wr, logits=None):
        self.x = x
        self.ws = self.ops.route(x, Wr, logits=logits)
        return self.ops.local_counts(x.shape[0], self.ws)

    # phase 2 --------------------------------------------------------------
    def plan_and_dispatch(self, C_all: torch.Tensor):
        """C_all [R, m] gathered counts (device).  Returns send buffers + splits."""
        plan = self.ops.plan_counts(C_all)
        # one device-to-host copy (the forward's only synchronisation): counts + executor map
        m = self.pl.m
        both = torch.cat([C_all.reshape(-1).to(torch.int64), plan["exec_of_expert"].reshape(-1).to(torch.int64)])
        both = both.cpu().numpy()
        C_host = both[:-m].reshape(self.pl.R, m)
        exec_host = both[-m:]
        tabs = self.pl.tables(C_host, exec_host, rank=self.rank)
        dev = self.x.device
        T = self.x.shape[0]
        nrep = self.pl.nrep
        self.dtabs = self._upload_tables(tabs, dev)
        row_base = self.dtabs["row_base"]
        send_x = torch.empty(tabs["R_send"], self.d, dtype=self.dtype, device=dev)
        send_w = torch.empty(tabs["R_send"], dtype=torch.float32, device=dev)
        row_of = torch.empty(T * self.K * nrep, dtype=torch.int32, device=dev)
        self.ops.dispatch(T, row_base, nrep, self.x, send_x, send_w, row_of, workspace=self.ws)
        self.state = EPState(T=T, tabs=tabs, row_of=row_of, send_x=send_x, send_w=send_w)
        return send_x, send_w, tabs["send_splits"], tabs["recv_splits"]

    # phase 3 --------------------------------------------------------------
    timers = None   # optional [start, end] torch.cuda.Event pair recorded around the local grouped FFN

    def compute(self, recv_x, recv_w):
        tb = self.state.tabs
        dev = recv_x.device
        eo = np.asarray(tb["exec_off"])
        rows = np.diff(eo)
        n_o = tb["n_orig"]
        self.last_ffn_flops = 6.0 * self.d * (self.pl.f * rows[:n_o].sum() + self.pl.f_u * rows[n_o:].sum())
        dt = self.dtabs   # device copies of this forward's tables (one upload in plan_and_dispatch)
        Rr = recv_x.shape[0]
        gx = torch.empty_like(recv_x)
        gw = torch.empty_like(recv_w)
        self.ops.block_copy(recv_x, gx, dt["fwd_src_off"], dt["fwd_dst_start"], recv_w, gw)
        h_buf = torch.empty(Rr, self.pl.f, dtype=self.dtype, device=dev)
        gy = torch.empty(Rr, self.d, dtype=self.dtype, device=dev)
        if self.timers is not None:
            self.timers[0].record()
        self.ops.expert_ffn(gx, gw, dt["exec_off"], dt["mtile_off"], tb["n_orig"], tb["n_united"],
                            self.pl.f_u, self.ex, self.un, h_buf, gy)
        if self.timers is not None:
            self.timers[1].record()
        ry = torch.empty_like(gy)
        self.ops.block_copy(gy, ry, dt["inv_src_off"], dt["inv_dst_start"])
        return ry

    # phase 4 --------------------------------------------------------------
    def combine(self, back_y, y=None):
        st = self.state
        if y is None:
            y = torch.empty_like(self.x)
        self.ops.combine(st.T, back_y, st.row_of, self.pl.nrep, self.x, y)
        return y

    # all phases with a real process group -----------------------------------
    def forward(self, x, Wr, comm: TorchComm, logits=None):
        cnt = self.route(x, Wr, logits)
        C_all = comm.all_gather_counts(cnt)
        send_x, send_w, s_split, r_split = self.plan_and_dispatch(C_all)
        recv_x = torch.empty(sum(r_split), self.d, dtype=self.dtype, device=x.device)
        recv_w = torch.empty(sum(r_split), dtype=torch.float32, device=x.device)
        comm.all_to_all(recv_x, send_x, r_split, s_split)
        comm.all_to_all(recv_w, send_w, r_split, s_split)
        ry = self.compute(recv_x, recv_w)
        back = torch.empty(sum(s_split), self.d, dtype=self.dtype, device=x.device)
        comm.all_to_all(back, ry, s_split, r_split)
        return self.combine(back)


def virtual_ep_forward(ranks, xs, Wr, logits=None):
    """Run an EP forward over len(ranks) logical ranks inside one process,
    emulating the collectives with tensor copies (single-GPU tests)."""
    R = len(ranks)
    cnts = [rk.route(x, Wr, None if logits is None else logits[i]) for i, (rk, x) in enumerate(zip(ranks, xs))]
    C_all = torch.stack([c.to(cnts[0].device) for c in cnts])
    outs = [rk.plan_and_dispatch(C_all) for rk in ranks]
    # all_to_all #1: rank q receives, in source order, segment q of every source
    recv = []
    for q in range(R):
        xs_q, ws_q = [], []
        for r in range(R):
            sx, sw, ss, _ = outs[r]
            o = sum(ss[:q])
            xs_q.append(sx[o:o + ss[q]])
            ws_q.append(sw[o:o + ss[q]])
        recv.append((torch.cat(xs_q), torch.cat(ws_q)))
    ry = [rk.compute(*recv[q]) for q, rk in enumerate(ranks)]
    # all_to_all #2: source r gets back, in destination order, its segment from every q
    ys = []
    for r in range(R):
        parts = []
        for q in range(R):
            rs = outs[q][3]          # recv splits of q (per source)
            o = sum(rs[:r])
            parts.append(ry[q][o:o + rs[r]])
        ys.append(ranks[r].combine(torch.cat(parts)))
    return ys
