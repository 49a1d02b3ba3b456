"""Expert-parallel (EP) brownout MoE forward over R ranks.

Binding of the library's EP API (include/brownout.h "Expert parallelism"):
argument marshalling only.  Placement, the global Alg. 1 plan, every exchange
table, the permutation, the grouped FFN and the combine run in libbrownout
(host placement in C++, everything per forward in CUDA kernels).  The three
exchanges of a forward are either

  * done by the library itself over its own NCCL communicator
    (EPContext.init_nccl + EPContext.forward: one call per forward; in padded
    mode no host synchronisation and CUDA-graph capturable), or
  * done by the caller between the stage calls (ep_forward_staged with a
    torch.distributed group - NCCL on GPUs, gloo in tests - or
    virtual_ep_forward, which emulates R ranks on one GPU with device copies).

Stages per forward on rank r (D18: one global plan over the concatenated batch):

  1. route     router + top-K + local counts -> count row [m + 4]    (kernels)
  2. all-gather of the count rows [R, m + 4]                          (exchange)
  3. dispatch  Alg. 1 on the column sums with rank 0's knob, exchange
               tables, permutation + gather into the send buffer     (kernels)
  4. all-to-all send -> recv (rows + gate weights)                    (exchange)
  5. compute   regroup by executor, grouped SwiGLU GEMMs x gate weight,
               back to the receive layout                             (kernels)
  6. all-to-all ret -> back                                           (exchange)
  7. combine   y_t = [x_t] + sum over slots and f-slices              (kernel)
"""
from __future__ import annotations

import ctypes as C

import torch

from .brownout import (BrownoutMoE, _check, _lib, _ptr, _stream, bo_ep_config, bo_ep_info, bo_ep_ws_layout)


def placement(m: int, way: int, f: int, world: int, rank: int) -> dict:
    """Static placement of one rank (host only): bo_ep_placement + slices."""
    info = bo_ep_info()
    _check(_lib.bo_ep_placement(m, way, f, world, rank, C.byref(info)))
    n = info.n_united_local
    g = (C.c_int32 * max(n, 1))()
    s = (C.c_int32 * max(n, 1))()
    _check(_lib.bo_ep_placement_slices(m, way, f, world, rank, g, s, max(n, 1)))
    out = {k: getattr(info, k) for k, _ in bo_ep_info._fields_}
    out["slices"] = [(int(g[i]), int(s[i])) for i in range(n)]
    return out


class EPContext:
    """One rank's EP context (bo_ep) on a BrownoutMoE handle."""

    def __init__(self, moe: BrownoutMoE, world: int, rank: int, max_tokens: int, padded: int = -1, device="cuda"):
        self.moe = moe
        cfg = bo_ep_config(world=world, rank=rank, padded=padded, max_tokens=max_tokens)
        h = C.c_void_p()
        _check(_lib.bo_ep_create(moe._h, C.byref(cfg), C.byref(h)))
        self._h = h
        info = bo_ep_info()
        _check(_lib.bo_ep_get_info(h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in bo_ep_info._fields_}
        self.world, self.rank = world, rank
        self.slices = placement(moe.cfg.num_experts, moe.cfg.way, moe.cfg.ffn, world, rank)["slices"]
        L = bo_ep_ws_layout()
        _check(_lib.bo_ep_workspace_layout(h, C.byref(L)))
        self.L = L
        self.ws = torch.empty(L.total_bytes, dtype=torch.uint8, device=device)
        self.T = 0

    def close(self):
        """bo_ep_destroy (also on garbage collection).  Destroy every CUDA graph that
        captured this context's forward first: such a graph holds the communicator's
        persistent NCCL resources, and destroying the communicator under it blocks."""
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.bo_ep_destroy(h)
            self._h = None

    def __del__(self):
        self.close()

    # -- static ---------------------------------------------------------------
    @property
    def padded(self) -> bool:
        return bool(self.info["padded"])

    @property
    def cap(self) -> int:
        return int(self.info["cap"])

    def local_weights(self, experts, united):
        """This rank's weights: originals [e0, e1) (views) and its united f-slices,
        stacked in executor order (copies; once per weight load)."""
        Wg, Wu, Wd = experts
        e0, e1, fu = self.info["e0"], self.info["e1"], self.info["f_united"]
        ex = (Wg[e0:e1], Wu[e0:e1], Wd[e0:e1]) if e1 > e0 else None
        if not self.slices or united is None:
            return ex, None
        UWg, UWu, UWd = united
        ug = torch.stack([UWg[j, s * fu:(s + 1) * fu, :] for j, s in self.slices]).contiguous()
        uu = torch.stack([UWu[j, s * fu:(s + 1) * fu, :] for j, s in self.slices]).contiguous()
        ud = torch.stack([UWd[j, :, s * fu:(s + 1) * fu] for j, s in self.slices]).contiguous()
        return ex, (ug, uu, ud)

    # -- workspace views --------------------------------------------------------
    def _view(self, off, n, dt):
        nbytes = n * torch.tensor([], dtype=dt).element_size()
        return self.ws[off:off + nbytes].view(dt)

    def count_row(self):
        return self._view(self.L.count_row, self.moe.cfg.num_experts + 4, torch.int32)

    def gathered(self):
        return self._view(self.L.gathered, self.world * (self.moe.cfg.num_experts + 4), torch.int32)

    def rows(self, name):
        """send / recv exchange rows [rows_max, d] (back aliases send, ret aliases recv)."""
        d, n = self.moe.cfg.hidden, int(self.L.rows_max)
        return self._view(getattr(self.L, name), n * d, self.moe.torch_dtype).view(n, d)

    def weights(self, name):
        return self._view(getattr(self.L, name + "_w"), int(self.L.rows_max), torch.float32)

    def tables(self):
        """Device views of this forward's exchange tables (include/brownout.h order)."""
        m, R = self.moe.cfg.num_experts, self.world
        nl, nrep = self.info["n_local"], self.info["nrep"]
        nb = nl * R
        sizes = (("row_base", m * nrep), ("send_rows", R), ("recv_rows", R), ("fwd_dst", nb + 1), ("fwd_len", nb),
                 ("fwd_src", nb), ("inv_dst", nb + 1), ("inv_len", nb), ("inv_src", nb), ("exec_off", nl + 1),
                 ("mtile_off", nl + 1), ("totals", 2))
        flat = self._view(self.L.tables, sum(n for _, n in sizes), torch.int32)
        out, o = {}, 0
        for k, n in sizes:
            out[k] = flat[o:o + n]
            o += n
        return out

    def local_rows(self):
        """Rows each local executor processed in the last forward (host read, synchronises)."""
        eo = self.tables()["exec_off"].cpu().tolist()
        return [b - a for a, b in zip(eo[:-1], eo[1:])]

    def plan(self):
        m = self.moe.cfg.num_experts
        return {"exec_of_expert": self._view(self.L.exec_of_expert, m, torch.int32),
                "counts": self._view(self.L.counts, m, torch.int32),
                "stats": self._view(self.L.stats, 8, torch.int64)}

    # -- library-owned NCCL ------------------------------------------------------
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(_lib.bo_ep_nccl_unique_id(buf))
        return bytes(buf)

    def init_nccl(self, uid: bytes):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        _check(_lib.bo_ep_init(self._h, buf))

    def forward(self, x, Wr, local_experts, local_united, y=None, stream=None):
        """The whole EP forward over the library's communicator (after init_nccl)."""
        ex = local_experts or (None, None, None)
        un = local_united or (None, None, None)
        if y is None:
            y = torch.empty_like(x)
        _check(_lib.bo_ep_forward(self._h, _ptr(x), x.shape[0], _ptr(Wr), *[_ptr(w) for w in ex],
                                  *[_ptr(w) for w in un], _ptr(y), _ptr(self.ws), self.ws.numel(), _stream(stream)))
        return y

    # -- stages --------------------------------------------------------------------
    def route(self, x, Wr, logits=None, stream=None):
        self.T = x.shape[0]
        _check(_lib.bo_ep_route(self._h, _ptr(x), x.shape[0], _ptr(Wr), _ptr(logits), _ptr(self.ws), self.ws.numel(),
                                _stream(stream)))
        return self.count_row()

    def dispatch(self, x, stream=None):
        _check(_lib.bo_ep_dispatch(self._h, _ptr(x), _ptr(self.ws), self.ws.numel(), _stream(stream)))

    def splits(self, stream=None):
        """(send_rows[q], recv_rows[r]): exact mode reads them from the device
        (one stream synchronisation); padded mode returns cap for every peer."""
        s = (C.c_int64 * self.world)()
        r = (C.c_int64 * self.world)()
        _check(_lib.bo_ep_splits(self._h, _ptr(self.ws), self.ws.numel(), s, r, _stream(stream)))
        return [int(v) for v in s], [int(v) for v in r]

    def compute(self, local_experts, local_united, stream=None):
        ex = local_experts or (None, None, None)
        un = local_united or (None, None, None)
        _check(_lib.bo_ep_compute(self._h, *[_ptr(w) for w in ex], *[_ptr(w) for w in un], _ptr(self.ws),
                                  self.ws.numel(), _stream(stream)))

    def combine(self, x, y=None, stream=None):
        if y is None:
            y = torch.empty_like(x)
        _check(_lib.bo_ep_combine(self._h, _ptr(x), _ptr(y), _ptr(self.ws), self.ws.numel(), _stream(stream)))
        return y


class TorchComm:
    """Exchange over a torch.distributed process group (NCCL on GPUs, gloo in tests)."""

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

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor):
        o = self._host(out)
        self.dist.all_gather_into_tensor(o, self._host(inp.contiguous()), group=self.group)
        if o is not out:
            out.copy_(o)

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        o = self._host(out)
        self.dist.all_to_all_single(o, self._host(inp), output_split_sizes=list(out_splits),
                                    input_split_sizes=list(in_splits), group=self.group)
        if o is not out:
            out.copy_(o)


def ep_forward_staged(ctx: EPContext, x, Wr, local_experts, local_united, comm: TorchComm, logits=None):
    """One EP forward with the exchanges done by `comm` between the library stages."""
    row = ctx.route(x, Wr, logits)
    comm.all_gather(ctx.gathered(), row)
    ctx.dispatch(x)
    send, recv = ctx.splits()
    ns, nr = sum(send), sum(recv)
    comm.all_to_all(ctx.rows("recv")[:nr], ctx.rows("send")[:ns], recv, send)
    comm.all_to_all(ctx.weights("recv")[:nr], ctx.weights("send")[:ns], recv, send)
    ctx.compute(local_experts, local_united)
    comm.all_to_all(ctx.rows("send")[:ns], ctx.rows("recv")[:nr], send, recv)   # ret -> back
    return ctx.combine(x)


def virtual_ep_forward(ctxs, xs, Wr, weights, logits=None):
    """An EP forward over len(ctxs) logical ranks in one process: the exchanges
    are device copies between the contexts' workspaces (single-GPU tests).  In
    padded mode every copy has a fixed size, so the whole call can be captured
    in a CUDA graph (no host synchronisation anywhere)."""
    R = len(ctxs)
    rows = [c.route(x, Wr, None if logits is None else logits[i]) for i, (c, x) in enumerate(zip(ctxs, xs))]
    g = torch.stack(rows).reshape(-1)
    for c in ctxs:
        c.gathered().copy_(g)
    for c, x in zip(ctxs, xs):
        c.dispatch(x)
    sp = [c.splits() for c in ctxs]

    def seg(splits, q):
        return sum(splits[:q]), splits[q]

    for q in range(R):                       # all-to-all #1: recv_q[r's segment] = send_r[q's segment]
        for r in range(R):
            so, sn = seg(sp[r][0], q)
            ro, rn = seg(sp[q][1], r)
            assert sn == rn
            ctxs[q].rows("recv")[ro:ro + rn].copy_(ctxs[r].rows("send")[so:so + sn])
            ctxs[q].weights("recv")[ro:ro + rn].copy_(ctxs[r].weights("send")[so:so + sn])
    for c, (ex, un) in zip(ctxs, weights):
        c.compute(ex, un)
    for r in range(R):                       # all-to-all #2: back_r[q's segment] = ret_q[r's segment]
        for q in range(R):
            so, sn = seg(sp[r][0], q)
            ro, rn = seg(sp[q][1], r)
            ctxs[r].rows("send")[so:so + sn].copy_(ctxs[q].rows("recv")[ro:ro + rn])
    return [c.combine(x) for c, x in zip(ctxs, xs)]
