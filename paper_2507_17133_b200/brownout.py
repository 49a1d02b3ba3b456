"""ctypes binding of libbrownout.so (include/brownout.h).

Argument marshalling only: every step of the forward runs in the library's
CUDA kernels.  torch is used for device memory and streams.  If the shared
library is missing or fails to load, importing this module raises: there is
no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BO_LIB=probe loads the instrumentation build (build.py --variant probe); the product
# library otherwise.  Either way there is no fallback.
LIB_PATH = os.path.join(_HERE, "libbrownout.so" if os.environ.get("BO_LIB", "") != "probe"
                        else "libbrownout_probe.so")

BO_OK, BO_ERR_INVALID_ARG, BO_ERR_SHAPE, BO_ERR_UNSUPPORTED, BO_ERR_CUDA, BO_ERR_NCCL, BO_ERR_WORKSPACE = range(7)
BO_BF16, BO_FP32 = 0, 1
BO_PARTIAL, BO_FULL = 0, 1
BO_UNITED_MEAN = 0
# bo_engine_option (include/brownout.h): name -> id
ENGINE_OPTIONS = {n: i for i, n in enumerate((
    "cta_pairs", "pair_rows1", "pair_rows2", "tile_alt", "swap_tail", "decode_pair2", "gemm2_splitk",
    "fused_combine", "tma_store", "store_hint", "b_policy", "router_mma", "router_split", "pdl", "route_fused", "tail_split"))}

EXPORTED = (
    "bo_create", "bo_destroy", "bo_workspace_size", "bo_workspace_layout", "bo_build_united", "bo_set_shared_experts",
    "bo_set_engine_option", "bo_get_engine_option",
    "bo_set_brownout", "bo_get_brownout", "bo_moe_forward", "bo_moe_forward_ex", "bo_plan_from_counts",
    "bo_route", "bo_expert_ffn", "bo_combine",
    "bo_ep_placement", "bo_ep_placement_slices", "bo_ep_create", "bo_ep_destroy", "bo_ep_get_info",
    "bo_ep_workspace_layout", "bo_ep_nccl_unique_id", "bo_ep_init", "bo_ep_forward", "bo_ep_route",
    "bo_ep_dispatch", "bo_ep_splits", "bo_ep_compute", "bo_ep_combine",
    "bo_set_profile_events", "bo_last_launch_count", "bo_last_kernels", "bo_status_string", "bo_last_error", "bo_version",
    "bo_distill_workspace_layout", "bo_distill_prepare", "bo_distill_load_united", "bo_distill_step",
)


class bo_config(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("ffn", C.c_int32), ("num_experts", C.c_int32), ("top_k", C.c_int32),
                ("way", C.c_int32), ("dtype", C.c_int32), ("add_residual", C.c_int32), ("dedup_united", C.c_int32),
                ("num_shared", C.c_int32), ("max_tokens", C.c_int64)]


class bo_plan_stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("executors_accessed", "n_s1", "n_united", "n_singleton",
                                         "rows_original", "rows_united", "rows_dropped", "rows_total")]


STATS_FIELDS = [f[0] for f in bo_plan_stats._fields_]


class bo_ws_layout(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("total_bytes", "logits", "topk_id", "topk_w", "tile_cnt", "tile_base",
                                          "counts", "exec_of_expert", "expert_row_off", "exec_off", "mtile_off",
                                          "stats", "row_of", "row_tok", "row_w", "xp", "h", "yp", "partial",
                                          "tile_xcnt", "tile_xbase", "ksplit", "comb_cnt", "sk_part", "sk_flag")] + \
               [("T", C.c_int64), ("ntiles", C.c_int64), ("num_executors", C.c_int64)]


class bo_distill_layout(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("total_bytes", "hbar", "floor_", "loss", "xt", "teach_h", "teach_y", "p",
                                          "q", "hs", "hst", "y", "dy", "dyt", "dhs", "dpt", "dqt", "uwdt", "part",
                                          "off_tok", "off_teach", "off_f", "off_d")] + [("N", C.c_int64)]


class bo_ep_config(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("padded", C.c_int32), ("max_tokens", C.c_int64)]


class bo_ep_info(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("world", "rank", "padded", "e0", "e1", "n_united_local", "f_united", "nrep",
                                         "sliced", "n_exec", "n_local")] + [("cap", C.c_int64), ("rows_max", C.c_int64)]


class bo_ep_ws_layout(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("total_bytes", "route", "count_row", "gathered", "exec_of_expert",
                                          "expert_row_off", "plan_scratch", "stats", "counts", "tables", "splits",
                                          "send", "send_w", "recv", "recv_w", "grouped", "grouped_w", "h",
                                          "row_of")] + [("rows_max", C.c_int64)]


class BrownoutError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run paper_2507_17133_b200.build.build() "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    sig = {
        "bo_create": ([C.POINTER(bo_config), C.POINTER(vp)], C.c_int),
        "bo_destroy": ([vp], C.c_int),
        "bo_workspace_size": ([vp, i64, C.POINTER(C.c_size_t)], C.c_int),
        "bo_workspace_layout": ([vp, i64, C.POINTER(bo_ws_layout)], C.c_int),
        "bo_build_united": ([vp, vp, vp, vp, i32, vp, vp, vp, vp], C.c_int),
        "bo_set_engine_option": ([vp, i32, i32], C.c_int),
        "bo_get_engine_option": ([vp, i32, C.POINTER(i32)], C.c_int),
        "bo_set_brownout": ([vp, C.c_double, i32], C.c_int),
        "bo_set_shared_experts": ([vp, vp, vp, vp], C.c_int),
        "bo_get_brownout": ([vp, C.POINTER(C.c_double), C.POINTER(i32)], C.c_int),
        "bo_moe_forward": ([vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_moe_forward_ex": ([vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp, vp], C.c_int),
        "bo_plan_from_counts": ([vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "bo_route": ([vp, vp, i64, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_ep_placement": ([i32, i32, i32, i32, i32, C.POINTER(bo_ep_info)], C.c_int),
        "bo_ep_placement_slices": ([i32, i32, i32, i32, i32, vp, vp, i32], C.c_int),
        "bo_ep_create": ([vp, C.POINTER(bo_ep_config), C.POINTER(vp)], C.c_int),
        "bo_ep_destroy": ([vp], C.c_int),
        "bo_ep_get_info": ([vp, C.POINTER(bo_ep_info)], C.c_int),
        "bo_ep_workspace_layout": ([vp, C.POINTER(bo_ep_ws_layout)], C.c_int),
        "bo_ep_nccl_unique_id": ([vp], C.c_int),
        "bo_ep_init": ([vp, vp], C.c_int),
        "bo_ep_forward": ([vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_ep_route": ([vp, vp, i64, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_ep_dispatch": ([vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_ep_splits": ([vp, vp, C.c_size_t, vp, vp, vp], C.c_int),
        "bo_ep_compute": ([vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_ep_combine": ([vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_expert_ffn": ([vp, vp, i64, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "bo_combine": ([vp, i64, vp, vp, i32, vp, vp, vp], C.c_int),
        "bo_set_profile_events": ([vp, C.POINTER(vp), i32], C.c_int),
        "bo_distill_workspace_layout": ([vp, i64, C.POINTER(bo_distill_layout)], C.c_int),
        "bo_distill_prepare": ([vp, vp, i64, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_distill_load_united": ([vp, i64, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_distill_step": ([vp, vp, i64, C.c_float, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp], C.c_int),
        "bo_last_launch_count": ([vp], i32),
        "bo_last_kernels": ([vp], C.c_char_p),
        "bo_status_string": ([C.c_int], C.c_char_p),
        "bo_last_error": ([], C.c_char_p),
        "bo_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = _load()


def lib():
    return _lib


def _check(status: int):
    if status != BO_OK:
        raise BrownoutError(status, f"{_lib.bo_status_string(status).decode()}: {_lib.bo_last_error().decode()}")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _req(t, name, dtype, shape, device=None):
    """Argument check before a raw pointer crosses the ABI (the C side can only
    check alignment): dtype, contiguity, CUDA residency and shape."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


_TORCH_DTYPE = {BO_BF16: torch.bfloat16, BO_FP32: torch.float32}


class BrownoutMoE:
    """One MoE layer handle: bo_create / bo_set_brownout / bo_moe_forward."""

    def __init__(self, hidden, ffn, num_experts, top_k, way, dtype="bf16", add_residual=False,
                 max_tokens=16384, dedup=False, num_shared=0, **engine_options):
        self.cfg = bo_config(hidden=hidden, ffn=ffn, num_experts=num_experts, top_k=top_k, way=way,
                             dtype=BO_BF16 if dtype in ("bf16", torch.bfloat16) else BO_FP32,
                             add_residual=1 if add_residual else 0, dedup_united=1 if dedup else 0,
                             num_shared=num_shared, max_tokens=max_tokens)
        h = C.c_void_p()
        _check(_lib.bo_create(C.byref(self.cfg), C.byref(h)))
        self._h = h
        self.torch_dtype = _TORCH_DTYPE[self.cfg.dtype]
        self.G = -(-num_experts // way)
        self.E = num_experts + self.G
        self._ws = None
        for k, v in engine_options.items():
            self.set_option(k, v)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.bo_destroy(h)
            self._h = None

    # -- knob ------------------------------------------------------------
    def set_brownout(self, ratio: float, mode: str = "partial"):
        _check(_lib.bo_set_brownout(self._h, float(ratio), BO_FULL if mode == "full" else BO_PARTIAL))

    def get_brownout(self):
        r, m = C.c_double(), C.c_int32()
        _check(_lib.bo_get_brownout(self._h, C.byref(r), C.byref(m)))
        return r.value, ("full" if m.value == BO_FULL else "partial")

    # -- workspace -------------------------------------------------------
    def workspace_size(self, T: int) -> int:
        n = C.c_size_t()
        _check(_lib.bo_workspace_size(self._h, int(T), C.byref(n)))
        return n.value

    def workspace_layout(self, T: int) -> bo_ws_layout:
        L = bo_ws_layout()
        _check(_lib.bo_workspace_layout(self._h, int(T), C.byref(L)))
        return L

    def workspace(self, T: int, device="cuda") -> torch.Tensor:
        need = self.workspace_size(T)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=device)
        return self._ws

    # -- calls -----------------------------------------------------------
    def set_shared_experts(self, SWg, SWu, SWd):
        """Eq. 5 shared experts [N_s, f, d] / [N_s, d, f] (device tensors kept alive here)."""
        self._shared = (SWg, SWu, SWd)
        _check(_lib.bo_set_shared_experts(self._h, _ptr(SWg), _ptr(SWu), _ptr(SWd)))

    def build_united(self, Wg, Wu, Wd, stream=None):
        self._check_layer(torch.empty(0, self.cfg.hidden, dtype=self.torch_dtype, device=Wg.device),
                          None, (Wg, Wu, Wd), None)
        m, f, d = Wg.shape
        G = self.G
        UWg = torch.empty(G, f, d, dtype=Wg.dtype, device=Wg.device)
        UWu = torch.empty(G, f, d, dtype=Wu.dtype, device=Wu.device)
        UWd = torch.empty(G, d, f, dtype=Wd.dtype, device=Wd.device)
        _check(_lib.bo_build_united(self._h, _ptr(Wg), _ptr(Wu), _ptr(Wd), BO_UNITED_MEAN, _ptr(UWg), _ptr(UWu),
                                    _ptr(UWd), _stream(stream)))
        return UWg, UWu, UWd

    def set_option(self, name: str, value: int):
        """bo_set_engine_option: scheduling choice of the kernels (ENGINE_OPTIONS), never the result."""
        _check(_lib.bo_set_engine_option(self._h, ENGINE_OPTIONS[name], int(value)))

    def get_option(self, name: str) -> int:
        v = C.c_int32()
        _check(_lib.bo_get_engine_option(self._h, ENGINE_OPTIONS[name], C.byref(v)))
        return v.value

    def forward(self, x, Wr, experts, united, y=None, workspace=None, logits=None, stream=None, shared=None):
        """moe_forward(tokens, router, experts, united) -> y [T, d].
        shared: optional (SWg, SWu, SWd) for a handle created with num_shared > 0
        (same as calling set_shared_experts first)."""
        if shared is not None:
            self.set_shared_experts(*shared)
        T = x.shape[0]
        Wg, Wu, Wd = experts
        UWg, UWu, UWd = united if united is not None else (None, None, None)
        self._check_layer(x, Wr, experts, united, logits)
        if y is None:
            y = torch.empty_like(x)
        _req(y, "y", self.torch_dtype, x.shape, x.device)
        ws = workspace if workspace is not None else self.workspace(T, x.device)
        if logits is None:
            _check(_lib.bo_moe_forward(self._h, _ptr(x), T, _ptr(Wr), _ptr(Wg), _ptr(Wu), _ptr(Wd), _ptr(UWg),
                                       _ptr(UWu), _ptr(UWd), _ptr(y), _ptr(ws), ws.numel(), _stream(stream)))
        else:
            _check(_lib.bo_moe_forward_ex(self._h, _ptr(x), T, _ptr(Wr), _ptr(Wg), _ptr(Wu), _ptr(Wd), _ptr(UWg),
                                          _ptr(UWu), _ptr(UWd), _ptr(y), _ptr(ws), ws.numel(), _ptr(logits),
                                          _stream(stream)))
        return y

    def _check_layer(self, x, Wr, experts, united, logits=None):
        c, dt = self.cfg, self.torch_dtype
        d, f, m = c.hidden, c.ffn, c.num_experts
        _req(x, "x", dt, (x.shape[0], d))
        dev = x.device
        _req(Wr, "Wr", dt, (m, d), dev)
        if logits is not None:
            _req(logits, "logits", torch.float32, (x.shape[0], m), dev)
        if experts is not None:
            for name, t, shp in zip(("Wg", "Wu", "Wd"), experts, ((m, f, d), (m, f, d), (m, d, f))):
                _req(t, name, dt, shp, dev)
        if united is not None:
            for name, t, shp in zip(("UWg", "UWu", "UWd"), united, ((self.G, f, d), (self.G, f, d), (self.G, d, f))):
                _req(t, name, dt, shp, dev)

    def set_profile_events(self, events):
        """events: list of torch.cuda.Event(enable_timing=True) (>= launches + 1),
        recorded around every kernel of the following forwards (None entries skip
        that boundary); events=None disables."""
        if events is None:
            self._prof = None
            _check(_lib.bo_set_profile_events(self._h, None, 0))
            return
        for e in events:      # torch creates the underlying cudaEvent_t lazily, on first record
            if e is not None and not e.cuda_event:
                e.record()
        arr = (C.c_void_p * len(events))(*[C.c_void_p(e.cuda_event if e is not None else None) for e in events])
        self._prof = (events, arr)
        _check(_lib.bo_set_profile_events(self._h, arr, len(events)))

    def last_launch_count(self) -> int:
        return int(_lib.bo_last_launch_count(self._h))

    def last_kernels(self) -> list:
        """Names of the kernels the last forward launched, in launch order."""
        names = _lib.bo_last_kernels(self._h).decode()
        return names.split(",") if names else []

    def debug_arrays(self, T: int, workspace=None) -> dict:
        """Views of the workspace arrays of the last forward over T tokens."""
        ws = self._ws if workspace is None else workspace
        L = self.workspace_layout(T)
        m, K = self.cfg.num_experts, self.cfg.top_k
        d, f = self.cfg.hidden, self.cfg.ffn
        E = int(L.num_executors)            # m + G routed executors + N_s shared
        Ns = self.cfg.num_shared
        R = T * K + Ns * T
        eb = 2 if self.cfg.dtype == BO_BF16 else 4

        def view(off, n, dt):
            nbytes = n * torch.tensor([], dtype=dt).element_size()
            return ws[off:off + nbytes].view(dt)

        out = {
            "logits": view(L.logits, T * m, torch.float32).view(T, m),
            "topk_id": view(L.topk_id, T * K, torch.int32).view(T, K),
            "topk_w": view(L.topk_w, T * K, torch.float32).view(T, K),
            "counts": view(L.counts, m, torch.int32),
            "exec_of_expert": view(L.exec_of_expert, m, torch.int32),
            "expert_row_off": view(L.expert_row_off, m, torch.int32),
            "exec_off": view(L.exec_off, E + 1, torch.int32),
            "mtile_off": view(L.mtile_off, E + 1, torch.int32),
            "stats": view(L.stats, 8, torch.int64),
            "row_of": view(L.row_of, T * (K + Ns), torch.int32),   # [T, K + N_s]
            "row_tok": view(L.row_tok, R, torch.int32),
            "row_w": view(L.row_w, R, torch.float32),
            "xp": view(L.xp, R * d, self.torch_dtype).view(R, d),
            "h": view(L.h, R * f, self.torch_dtype).view(R, f),
            "yp": view(L.yp, R * d, self.torch_dtype).view(R, d),
        }
        del eb
        return out

    # -- expert-parallel building blocks (include/brownout.h) ----------------
    def route(self, x, Wr, logits=None, workspace=None, stream=None):
        """a1-a4 on a local batch; returns the workspace (counts etc. inside)."""
        T = x.shape[0]
        self._check_layer(x, Wr if logits is None else None, None, None, logits)
        ws = workspace if workspace is not None else self.workspace(T, x.device)
        _check(_lib.bo_route(self._h, _ptr(x), T, _ptr(Wr), _ptr(logits), _ptr(ws), ws.numel(), _stream(stream)))
        return ws

    def expert_ffn(self, rows, row_w, exec_off, mtile_off, n_orig, n_united, f_united, experts, united, h_buf, out,
                   stream=None):
        Wg, Wu, Wd = experts if experts is not None else (None, None, None)
        UWg, UWu, UWd = united if united is not None else (None, None, None)
        _check(_lib.bo_expert_ffn(self._h, _ptr(rows), rows.shape[0], _ptr(row_w), _ptr(exec_off), _ptr(mtile_off),
                                  n_orig, n_united, f_united, _ptr(Wg), _ptr(Wu), _ptr(Wd), _ptr(UWg), _ptr(UWu),
                                  _ptr(UWd), _ptr(h_buf), _ptr(out), _stream(stream)))

    def combine(self, T, rows, row_of, nrep, x, y, stream=None):
        _check(_lib.bo_combine(self._h, T, _ptr(rows), _ptr(row_of), nrep, _ptr(x), _ptr(y), _stream(stream)))

    def plan_from_counts(self, counts: torch.Tensor, stream=None):
        """Alg. 1 on device counts (int32 [m]) -> dict of device tensors."""
        m = self.cfg.num_experts
        dev = counts.device
        exec_of = torch.empty(m, dtype=torch.int32, device=dev)
        erow = torch.empty(m, dtype=torch.int32, device=dev)
        eoff = torch.empty(2 * (self.E + 1) + m, dtype=torch.int32, device=dev)
        stats = torch.empty(8, dtype=torch.int64, device=dev)
        _check(_lib.bo_plan_from_counts(self._h, _ptr(counts), _ptr(exec_of), _ptr(erow), _ptr(eoff), _ptr(stats),
                                        _stream(stream)))
        return {"exec_of_expert": exec_of, "expert_row_off": erow, "exec_off": eoff[:self.E + 1], "stats": stats}


class UnitedDistiller:
    """United-expert distillation (paper §4.2, Eq. 4; include/brownout.h
    bo_distill_*): trains the G united experts of `moe`'s layer against their
    groups' original experts on the token matrix X [N, d] (N % 64 == 0) by
    plain gradient descent on fp32 masters.  The bf16 united tensors returned
    by `united` are what BrownoutMoE.forward consumes."""

    def __init__(self, moe: BrownoutMoE, N: int, device="cuda"):
        self.moe = moe
        self.N = int(N)
        self.L = bo_distill_layout()
        _check(_lib.bo_distill_workspace_layout(moe._h, self.N, C.byref(self.L)))
        self.ws = torch.empty(self.L.total_bytes, dtype=torch.uint8, device=device)
        self.X = None
        self.masters = None
        self.united = None

    def prepare(self, X, Wg, Wu, Wd, stream=None):
        """Teacher outputs of every original expert on X, their group means and
        variance floors (once per token set)."""
        assert X.shape[0] == self.N
        self.X = X
        self._experts = (Wg, Wu, Wd)
        _check(_lib.bo_distill_prepare(self.moe._h, _ptr(X), self.N, _ptr(Wg), _ptr(Wu), _ptr(Wd), _ptr(self.ws),
                                       self.ws.numel(), _stream(stream)))

    def load_united(self, UWg, UWu, UWd, stream=None):
        """Initial student weights (bf16, e.g. BrownoutMoE.build_united); the
        tensors are then updated in place by every step."""
        self.united = (UWg, UWu, UWd)
        self.masters = tuple(torch.empty(u.shape, dtype=torch.float32, device=u.device) for u in self.united)
        _check(_lib.bo_distill_load_united(self.moe._h, self.N, *[_ptr(u) for u in self.united],
                                           *[_ptr(w) for w in self.masters], _ptr(self.ws), self.ws.numel(),
                                           _stream(stream)))

    def step(self, lr: float, stream=None):
        _check(_lib.bo_distill_step(self.moe._h, _ptr(self.X), self.N, float(lr), *[_ptr(w) for w in self.masters],
                                    *[_ptr(u) for u in self.united], _ptr(self.ws), self.ws.numel(),
                                    _stream(stream)))

    def _view(self, off, n, dt):
        nbytes = n * torch.tensor([], dtype=dt).element_size()
        return self.ws[off:off + nbytes].view(dt)

    def loss(self):
        """Eq. 4 per group (fp64) of the weights that entered the last step."""
        return self._view(self.L.loss, self.moe.G, torch.float64)

    def floor(self):
        return self._view(self.L.floor_, self.moe.G, torch.float64)

    def hbar(self):
        d = self.moe.cfg.hidden
        return self._view(self.L.hbar, self.moe.G * self.N * d, torch.float32).view(self.moe.G, self.N, d)
