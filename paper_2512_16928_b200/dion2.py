"""Thin ctypes binding over libdion2.so (include/dion2.h).

Argument marshalling only: every step of the Dion2 update runs in the CUDA
kernels behind the C ABI.  PyTorch supplies device memory and the current
stream.  There is no CPU fallback: if the extension is missing or a tensor is
not on a CUDA device, these functions raise.
"""
from __future__ import annotations

import collections
import ctypes
import os
from typing import Dict, List, Optional, Sequence, Tuple

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libdion2.so")

MAX_NS_STEPS = 16
AXIS = {"rows": 0, "cols": 1, "auto": 2}
PRECISION = {"bf16": 0, "fp32": 1}
SELECT = {"l1": 0, "random": 1}
NS_FORM = {"auto": 0, "direct": 1, "gram": 2}
ABI_VERSION = 7  # include/dion2.h DION2_ABI_VERSION
STATUS = {0: "OK", 1: "EINVAL_CONFIG", 2: "EINVAL_SHAPE", 3: "EWORKSPACE", 4: "EUNSUPPORTED",
          5: "ECUDA", 6: "ENCCL", 7: "ENONFINITE"}
EXPORTED = ["dion2_config_init", "dion2_workspace_size", "dion2_step", "dion2_step_batched", "dion2_get_status",
            "dion2_strerror", "dion2_set_phase_timing", "dion2_get_phase_times", "dion2_phase_name",
            "dion2_last_launch_count", "dion2_abi_version", "dion2_dist_info", "dion2_step_batched_dist",
            "dion2_step_batched_loopback", "dion2_dpsync_workspace_size", "dion2_step_batched_dpsync",
            "dion2_step_batched_dpsync_loopback", "dion2_release_workspace", "dion2_dist_exchange_mode"]


class Dion2Matrix(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("W", ctypes.c_void_p), ("M", ctypes.c_void_p), ("G", ctypes.c_void_p),
                ("sel_out", ctypes.c_void_p), ("O_out", ctypes.c_void_p),
                ("m_transposed", ctypes.c_int32), ("storage_transposed", ctypes.c_int32), ("ldm", ctypes.c_int64)]


class Dion2Config(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_float), ("mu", ctypes.c_float), ("lr", ctypes.c_float),
                ("ns_steps", ctypes.c_int32), ("ns_coeffs", (ctypes.c_float * 3) * MAX_NS_STEPS),
                ("ns_eps", ctypes.c_float), ("axis", ctypes.c_int32), ("select", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("grad_dtype", ctypes.c_int32), ("decay_mode", ctypes.c_int32),
                ("scale_mode", ctypes.c_int32), ("seed", ctypes.c_uint64), ("step", ctypes.c_uint64),
                ("ns_form", ctypes.c_int32), ("reserved0", ctypes.c_int32), ("w_dtype", ctypes.c_int32)]


class Dion2Shard(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("cols", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("W", ctypes.c_void_p), ("M", ctypes.c_void_p), ("G", ctypes.c_void_p), ("sel_out", ctypes.c_void_p),
                ("m_transposed", ctypes.c_int32), ("reserved", ctypes.c_int32), ("ldm", ctypes.c_int64)]


class Dion2Error(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)} ({_lib().dion2_strerror(code).decode()})")


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libdion2.so not built ({LIB_PATH}); run python -m paper_2512_16928_b200._build")
        lib = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        lib.dion2_config_init.argtypes = [P(Dion2Config)]
        lib.dion2_workspace_size.argtypes = [P(Dion2Matrix), ctypes.c_int32, P(Dion2Config), P(ctypes.c_size_t)]
        lib.dion2_step.argtypes = [P(Dion2Matrix), P(Dion2Config), ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        lib.dion2_step_batched.argtypes = [P(Dion2Matrix), ctypes.c_int32, P(Dion2Config), ctypes.c_void_p,
                                           ctypes.c_size_t, ctypes.c_void_p]
        lib.dion2_get_status.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(ctypes.c_int32)]
        lib.dion2_release_workspace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        lib.dion2_release_workspace.restype = ctypes.c_int32
        lib.dion2_strerror.argtypes = [ctypes.c_int]
        lib.dion2_strerror.restype = ctypes.c_char_p
        lib.dion2_set_phase_timing.argtypes = [ctypes.c_int32]
        lib.dion2_get_phase_times.argtypes = [P(ctypes.c_float), P(ctypes.c_int32), ctypes.c_int32, P(ctypes.c_int32)]
        lib.dion2_phase_name.argtypes = [ctypes.c_int32]
        lib.dion2_phase_name.restype = ctypes.c_char_p
        lib.dion2_last_launch_count.restype = ctypes.c_int32
        lib.dion2_abi_version.restype = ctypes.c_int32
        if lib.dion2_abi_version() != ABI_VERSION:
            raise RuntimeError(f"libdion2.so ABI {lib.dion2_abi_version()} != binding ABI {ABI_VERSION}; rebuild it")
        I32, I64 = P(ctypes.c_int32), P(ctypes.c_int64)
        lib.dion2_dist_info.argtypes = [P(Dion2Shard), ctypes.c_int32, P(Dion2Config), ctypes.c_int32, ctypes.c_int32,
                                        I32, I32, I64, I64, I64, I64, P(ctypes.c_size_t)]
        lib.dion2_step_batched_dist.argtypes = [P(Dion2Shard), ctypes.c_int32, P(Dion2Config), ctypes.c_void_p,
                                                ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                                ctypes.c_void_p, P(ctypes.c_uint64)]
        lib.dion2_step_batched_loopback.argtypes = [P(Dion2Shard), ctypes.c_int32, P(Dion2Config),
                                                    P(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_int32,
                                                    ctypes.c_void_p, P(ctypes.c_uint64)]
        lib.dion2_dpsync_workspace_size.argtypes = [P(Dion2Matrix), ctypes.c_int32, P(Dion2Config), ctypes.c_int32,
                                                    P(ctypes.c_size_t)]
        lib.dion2_step_batched_dpsync.argtypes = [P(Dion2Matrix), ctypes.c_int32, P(Dion2Config), ctypes.c_void_p,
                                                  ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                                  ctypes.c_void_p, P(ctypes.c_uint64)]
        lib.dion2_dist_exchange_mode.argtypes = [ctypes.c_void_p]
        lib.dion2_step_batched_dpsync_loopback.argtypes = [P(Dion2Matrix), ctypes.c_int32, P(Dion2Config),
                                                           P(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_int32,
                                                           ctypes.c_void_p, P(ctypes.c_uint64)]
        _LIB = lib
    return _LIB


def make_config(alpha: float = 0.25, mu: float = 0.95, lr: float = 0.02, ns_steps: int = 5,
                ns_coeffs: Optional[Sequence[Tuple[float, float, float]]] = None, ns_eps: float = 1e-7,
                axis: str = "auto", precision: str = "bf16", grad_dtype: Optional[torch.dtype] = None,
                decay_mode: int = 0, scale_mode: int = 0, select: str = "l1", seed: int = 0,
                step: int = 0, ns_form: str = "auto", lr_device: bool = False,
                w_dtype: Optional[torch.dtype] = None, dist_direct: bool = False) -> Dion2Config:
    """ns_form: "auto" | "direct" | "gram" -- how the tensor-core Newton-Schulz map is evaluated
    (include/dion2.h dion2_ns_form, readings R23, R24).  w_dtype: torch.bfloat16 for
    bf16 weights (the update is computed in fp32 and rounded once), else fp32.  dist_direct:
    the distributed step's pieces travel by direct peer stores / loads (K3 pushes into the
    owner's receive window, K7 pulls from its outgoing window; NCCL symmetric memory) instead
    of NCCL send / recv (DION2_FLAG_DIST_DIRECT)."""
    cfg = Dion2Config()
    _lib().dion2_config_init(ctypes.byref(cfg))
    cfg.alpha, cfg.mu, cfg.lr, cfg.ns_steps, cfg.ns_eps = alpha, mu, lr, ns_steps, ns_eps
    if ns_coeffs is not None:
        if len(ns_coeffs) != ns_steps:
            raise ValueError("ns_coeffs must have ns_steps rows")
        for t, (a, b, c) in enumerate(ns_coeffs):
            cfg.ns_coeffs[t][0], cfg.ns_coeffs[t][1], cfg.ns_coeffs[t][2] = a, b, c
    cfg.axis = AXIS[axis]
    cfg.precision = PRECISION[precision]
    cfg.grad_dtype = 1 if grad_dtype == torch.bfloat16 else 0
    cfg.w_dtype = 1 if w_dtype == torch.bfloat16 else 0
    cfg.decay_mode, cfg.scale_mode = decay_mode, scale_mode
    cfg.select = SELECT[select]
    cfg.seed, cfg.step = seed, step
    cfg.ns_form = NS_FORM[ns_form]
    cfg.reserved0 = (1 if lr_device else 0) | (2 if dist_direct else 0)  # DION2_FLAG_LR_DEVICE | _DIST_DIRECT
    return cfg


def _ld(t: torch.Tensor) -> int:
    """Row stride in elements; a one-row tensor's stride(0) is arbitrary in torch (size-1 dims),
    its leading dimension is its width."""
    return t.stride(0) if t.shape[0] > 1 else t.shape[1]


def _check_tensor(t: torch.Tensor, name: str, dtype: torch.dtype, like: Optional[torch.Tensor] = None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.dim() != 2 or (t.stride(1) != 1 and t.shape[1] > 1):
        raise ValueError(f"{name} must be 2-D with unit column stride")
    if like is not None and (t.shape != like.shape or _ld(t) != _ld(like)):
        raise ValueError(f"{name} must match W's shape and row stride")


def describe(Ws: Sequence[torch.Tensor], Ms: Sequence[torch.Tensor], Gs: Sequence[torch.Tensor],
             sel_out: Optional[Sequence[Optional[torch.Tensor]]] = None,
             O_out: Optional[Sequence[Optional[torch.Tensor]]] = None,
             m_transposed: Optional[Sequence[bool]] = None,
             storage_transposed: Optional[Sequence[bool]] = None):
    """m_transposed[i]: M[i] is stored transposed relative to W[i] (column-mode matrices).
    storage_transposed[i]: W[i], M[i], G[i] hold the logical m x n matrix transposed, i.e. the
    tensors have shape (n, m) = (fan-in, fan-out) as JAX / Flax (in, out) kernels do; the
    axis, k and the sqrt(fan-out / fan-in) scale follow the logical shape."""
    n = len(Ws)
    if not (len(Ms) == n and len(Gs) == n) or n == 0:
        raise ValueError("Ws, Ms, Gs must be non-empty and equally long")
    arr = (Dion2Matrix * n)()
    gdt = Gs[0].dtype
    for i, (W, M, G) in enumerate(zip(Ws, Ms, Gs)):
        _check_tensor(W, "W", Ws[0].dtype)
        if W.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("W must be float32 or bfloat16")
        mt = bool(m_transposed[i]) if m_transposed is not None else False
        stt = bool(storage_transposed[i]) if storage_transposed is not None else False
        arr[i].storage_transposed = 1 if stt else 0
        if mt:
            _check_tensor(M, "M (transposed)", torch.float32)
            if tuple(M.shape) != (W.shape[1], W.shape[0]):
                raise ValueError("a transposed M must have shape (cols, rows)")
            arr[i].m_transposed, arr[i].ldm = 1, _ld(M)
        else:
            _check_tensor(M, "M", torch.float32, W)
        _check_tensor(G, "G", gdt, W)
        # rows / cols are the LOGICAL fan-out / fan-in (the tensor is (n, m) under storage_transposed)
        arr[i].rows, arr[i].cols = (W.shape[1], W.shape[0]) if stt else (W.shape[0], W.shape[1])
        arr[i].ld = _ld(W)
        arr[i].W, arr[i].M, arr[i].G = W.data_ptr(), M.data_ptr(), G.data_ptr()
        s = sel_out[i] if sel_out is not None else None
        o = O_out[i] if O_out is not None else None
        arr[i].sel_out = s.data_ptr() if s is not None else None
        arr[i].O_out = o.data_ptr() if o is not None else None
    return arr, gdt


def workspace_bytes(shapes: Sequence[Tuple[int, int]], **cfg_kw) -> int:
    n = len(shapes)
    arr = (Dion2Matrix * n)()
    for i, (m, nn) in enumerate(shapes):
        arr[i].rows, arr[i].cols, arr[i].ld = m, nn, nn
    cfg = make_config(**cfg_kw)
    out = ctypes.c_size_t(0)
    rc = _lib().dion2_workspace_size(arr, n, ctypes.byref(cfg), ctypes.byref(out))
    if rc:
        raise Dion2Error(rc, "dion2_workspace_size")
    return out.value


class Dion2:
    """Stateful convenience wrapper: caches the config and a workspace tensor.

    opt = Dion2(alpha=0.25); opt.step(Ws, Ms, Gs)   # all on one CUDA device
    """

    def __init__(self, m_transposed=None, storage_transposed=None, cuda_graph: bool = False, **cfg_kw):
        """m_transposed / storage_transposed: default per-matrix layout flags used by step()
        (see describe()).  cuda_graph: a step whose tensors and config repeat the previous call's
        runs eagerly and is captured once into a CUDA graph; later steps with that key replay
        it (no per-step host work, no launch gaps).  A key seen once (e.g. under a learning-rate
        schedule) just runs eagerly.  One call is always exactly one optimizer step."""
        self.cfg_kw = dict(cfg_kw)
        self.m_transposed = m_transposed
        self.storage_transposed = storage_transposed
        self.cuda_graph = cuda_graph
        self._graphs = collections.OrderedDict()  # key -> (graph, workspace slot), LRU order
        self._ws: Optional[torch.Tensor] = None

    # Graph mode: each captured tensor set gets its own library plan, selected by a workspace
    # base offset (the plan cache is keyed by the workspace pointer): a plan's device descriptor
    # table then holds that set's pointers for good, so replaying one graph after another
    # set's step cannot read another set's pointers.  The scratch itself is shared (graphs
    # run in stream order).
    GRAPH_SLOTS = 16
    SLOT_BYTES = 4096

    def workspace(self, arr, n, cfg, device) -> torch.Tensor:
        need = ctypes.c_size_t(0)
        rc = _lib().dion2_workspace_size(arr, n, ctypes.byref(cfg), ctypes.byref(need))
        if rc:
            raise Dion2Error(rc, "dion2_workspace_size")
        if self.cuda_graph:
            need.value += (self.GRAPH_SLOTS + 1) * self.SLOT_BYTES  # + the slot of uncaptured steps
        if self._ws is None or self._ws.numel() < need.value or self._ws.device != device:
            self._graphs.clear()  # captured graphs reference the old workspace
            self._release()
            self._ws = torch.empty(need.value, dtype=torch.uint8, device=device)
        return self._ws

    def _release(self) -> None:
        """Drop the library's plans (and their device tables) keyed on this object's workspace."""
        if self._ws is not None:
            _lib().dion2_release_workspace(self._ws.data_ptr(), self._ws.numel())
            self._ws = None

    def __del__(self):
        try:
            self._graphs.clear()
            self._release()
        except Exception:  # interpreter shutdown: the library may already be gone
            pass

    def step(self, Ws, Ms, Gs, sel_out=None, O_out=None, stream: Optional[torch.cuda.Stream] = None,
             m_transposed=None, storage_transposed=None, **override):
        self._last_sub = None
        self._last_stream = None
        if self.cuda_graph and stream is None:
            ptrs = lambda ts: tuple((t.data_ptr(), tuple(t.shape), tuple(t.stride()), t.dtype) if t is not None  # noqa: E731
                                    else None for t in ts)
            key = (ptrs(Ws), ptrs(Ms), ptrs(Gs), ptrs(sel_out or ()), ptrs(O_out or ()),
                   tuple(m_transposed if m_transposed is not None else self.m_transposed or ()),
                   tuple(storage_transposed if storage_transposed is not None else self.storage_transposed or ()),
                   # eta is not part of the key: the graph reads it from the workspace word
                   # (DION2_FLAG_LR_DEVICE), so a learning-rate schedule replays one graph
                   tuple(sorted((k, repr(v)) for k, v in {**self.cfg_kw, **override}.items() if k != "lr")),
                   torch.cuda.current_device())
            lr = float({**self.cfg_kw, **override}.get("lr", 0.02))
            hit = self._graphs.get(key)
            if hit is not None and self._ws is not None:
                self._graphs.move_to_end(key)
                self._write_lr(hit[1], lr)
                hit[0].replay()
                self._last_slot = hit[1]
                return
            prev, self._prev_key = getattr(self, "_prev_key", None), key
            if key != prev:
                # first call with this key: eager, in the slot reserved for uncaptured steps (a
                # config that changes every step, e.g. the random-selection counter, never captures)
                self._step(Ws, Ms, Gs, sel_out, O_out, None, m_transposed, storage_transposed, self.GRAPH_SLOTS,
                           lr_device=True, write_lr=lr, **override)
                return
            used = {slot for (_, slot) in self._graphs.values()}
            free = [i for i in range(self.GRAPH_SLOTS) if i not in used]
            if not free:  # evict the least recently replayed graph and reuse its slot
                _, (_, slot) = self._graphs.popitem(last=False)
                free = [slot]
            slot = free[0]
            self._step(Ws, Ms, Gs, sel_out, O_out, None, m_transposed, storage_transposed, slot, lr_device=True,
                       write_lr=lr, **override)
            ws_before = self._ws
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):  # captured, not executed: this call's step ran above
                self._step(Ws, Ms, Gs, sel_out, O_out, None, m_transposed, storage_transposed, slot, lr_device=True,
                           **override)
            if self._ws is ws_before:  # a reallocated workspace invalidated every graph (cleared)
                self._graphs[key] = (g, slot)
            return
        # an explicit stream in graph mode runs eagerly in the uncaptured slot: slot 0 may belong to
        # a captured graph, whose plan's descriptor table must keep that graph's pointers
        self._step(Ws, Ms, Gs, sel_out, O_out, stream, m_transposed, storage_transposed,
                   self.GRAPH_SLOTS if self.cuda_graph else 0, **override)
        self._last_stream = stream

    def _write_lr(self, slot: int, lr: float) -> None:
        """eta into the fp32 word at byte 8 of the slot's 4096-aligned workspace base (stream-ordered)."""
        base = self._ws.data_ptr()
        aligned = (base + slot * self.SLOT_BYTES + 4095) & ~4095
        off = aligned - base + 8
        self._ws[off:off + 4].view(torch.float32).fill_(lr)

    def _step(self, Ws, Ms, Gs, sel_out, O_out, stream, m_transposed, storage_transposed, slot,
              lr_device: bool = False, write_lr: Optional[float] = None, **override):
        kw = dict(self.cfg_kw)
        kw.update(override)
        kw["lr_device"] = lr_device
        if m_transposed is None:
            m_transposed = self.m_transposed
        if storage_transposed is None:
            storage_transposed = self.storage_transposed
        arr, gdt = describe(Ws, Ms, Gs, sel_out, O_out, m_transposed, storage_transposed)
        kw.setdefault("grad_dtype", gdt)
        kw.setdefault("w_dtype", Ws[0].dtype)
        cfg = make_config(**kw)
        dev = Ws[0].device
        ws = self.workspace(arr, len(Ws), cfg, dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        off = slot * self.SLOT_BYTES
        self._last_slot = slot
        if write_lr is not None:
            self._write_lr(slot, write_lr)
        rc = _lib().dion2_step_batched(arr, len(Ws), ctypes.byref(cfg), ws.data_ptr() + off, ws.numel() - off,
                                       st.cuda_stream)
        if rc:
            raise Dion2Error(rc, "dion2_step_batched")

    def step_host(self, Ws, Ms, Gs, G_host, sel_out=None, chunks: Optional[int] = None):
        """One optimizer step whose gradients arrive from the host: G_host[i] is a pinned CPU
        tensor copied into the device buffer Gs[i].  The matrices are split into `chunks`
        (default 8, env DION2_HOST_CHUNKS; measured e2e 90.1 / 89.0 / 88.5 ms for 2 / 4 / 8 on the
        1B set) contiguous groups of about equal parameter count; a side stream copies group c + 1
        while group c steps on the current stream, so the step hides under the host-to-device
        transfer.  Each group is its own batched library call (its own plan and workspace)."""
        n = len(Ws)
        if not (len(Ms) == n and len(Gs) == n and len(G_host) == n):
            raise ValueError("Ws, Ms, Gs, G_host must be equally long")
        for g, h in zip(Gs, G_host):
            if h.is_cuda or h.shape != g.shape or h.dtype != g.dtype:
                raise ValueError("G_host[i] must be a CPU tensor shaped and typed like Gs[i]")
        if chunks is None:
            chunks = int(os.environ.get("DION2_HOST_CHUNKS", "8"))
        sizes = [w.numel() for w in Ws]
        total, bounds, acc, c0 = sum(sizes), [], 0, 0
        chunks = max(1, min(chunks, n))
        for i, sz in enumerate(sizes):
            acc += sz
            if len(bounds) < chunks - 1 and acc * chunks >= total * (len(bounds) + 1) and i + 1 < n:
                bounds.append((c0, i + 1))
                c0 = i + 1
        bounds.append((c0, n))
        key = tuple(bounds)
        if getattr(self, "_host_key", None) != key:
            mt = self.m_transposed
            self._host_subs = [Dion2(m_transposed=list(mt[a:b]) if mt is not None else None,
                                     storage_transposed=list(self.storage_transposed[a:b])
                                     if self.storage_transposed is not None else None,
                                     cuda_graph=self.cuda_graph, **self.cfg_kw) for (a, b) in bounds]
            self._host_key = key
            self._copy_stream = torch.cuda.Stream(device=Ws[0].device)
        for sub in self._host_subs:  # the config may have changed since the subs were made
            sub.cfg_kw = dict(self.cfg_kw)
        cur = torch.cuda.current_stream(Ws[0].device)
        cs = self._copy_stream
        cs.wait_stream(cur)  # the previous step has finished reading the G buffers
        events = []
        with torch.cuda.stream(cs):
            for (a, b) in bounds:
                for i in range(a, b):
                    Gs[i].copy_(G_host[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                events.append(ev)
        for (a, b), ev, sub in zip(bounds, events, self._host_subs):
            cur.wait_event(ev)
            sub.step(Ws[a:b], Ms[a:b], Gs[a:b], sel_out=list(sel_out[a:b]) if sel_out is not None else None)
        self._last_sub = self._host_subs

    def status(self) -> Tuple[int, int]:
        if getattr(self, "_last_sub", None):
            worst, bad = 0, -1
            for sub, (a, _) in zip(self._last_sub, self._host_key):
                rc, b = sub.status()
                if rc and bad < 0:
                    worst, bad = rc, a + b
            return worst, bad
        bad = ctypes.c_int32(-1)
        ws = self._ws.data_ptr() + getattr(self, "_last_slot", 0) * self.SLOT_BYTES if self._ws is not None else None
        st = getattr(self, "_last_stream", None) or torch.cuda.current_stream()
        rc = _lib().dion2_get_status(ws, st.cuda_stream, ctypes.byref(bad))
        return rc, bad.value


def step(W, M, G, **kw):
    """One Dion2 step on one matrix (dion2_step)."""
    Dion2(**kw).step([W], [M], [G])


def set_phase_timing(enable: bool) -> None:
    _lib().dion2_set_phase_timing(1 if enable else 0)


def get_phase_times() -> Dict[str, Tuple[float, int]]:
    cap = 16
    ms = (ctypes.c_float * cap)()
    cnt = (ctypes.c_int32 * cap)()
    n = ctypes.c_int32(0)
    rc = _lib().dion2_get_phase_times(ms, cnt, cap, ctypes.byref(n))
    if rc:
        raise Dion2Error(rc, "dion2_get_phase_times")
    return {_lib().dion2_phase_name(i).decode(): (ms[i], cnt[i]) for i in range(n.value)}


def last_launch_count() -> int:
    return int(_lib().dion2_last_launch_count())


# ----------------------------------------------------------------------------------- multi-GPU
def _shards(shapes, Ws=None, Ms=None, Gs=None, sels=None, m_transposed=None):
    """m_transposed[i]: the local M shard is stored transposed, shape (shard cols, shard rows)."""
    n = len(shapes)
    arr = (Dion2Shard * n)()
    for i, (m, nn) in enumerate(shapes):
        arr[i].rows, arr[i].cols = m, nn
        mt = bool(m_transposed[i]) if m_transposed is not None else False
        arr[i].m_transposed = 1 if mt else 0
        arr[i].ldm = 1 << 40
        if Ws is not None:
            W = Ws[i]
            _check_tensor(W, "W shard", Ws[0].dtype)
            if W.dtype not in (torch.float32, torch.bfloat16):
                raise ValueError("W shard must be float32 or bfloat16")
            if mt:
                _check_tensor(Ms[i], "M shard (transposed)", torch.float32)
                if tuple(Ms[i].shape) != (W.shape[1], W.shape[0]):
                    raise ValueError("a transposed M shard must have shape (shard cols, shard rows)")
                arr[i].ldm = _ld(Ms[i])
            else:
                _check_tensor(Ms[i], "M shard", torch.float32, W)
            _check_tensor(Gs[i], "G shard", Gs[0].dtype, W)
            arr[i].ld = _ld(W)
            arr[i].W, arr[i].M, arr[i].G = W.data_ptr(), Ms[i].data_ptr(), Gs[i].data_ptr()
            s = sels[i] if sels is not None else None
            arr[i].sel_out = s.data_ptr() if s is not None else None
        else:
            arr[i].ld = 1 << 40
    return arr


def dist_info(shapes: Sequence[Tuple[int, int]], world: int, rank: int, m_transposed=None, **cfg_kw) -> dict:
    """Host-only layout of the owner-compute step (dion2_dist_info): per matrix the
    resolved axis, owner rank and local shard shape; per peer the bytes sent/received in
    one exchange direction; this rank's workspace size."""
    n = len(shapes)
    arr = _shards(shapes, m_transposed=m_transposed)
    cfg = make_config(**cfg_kw)
    ax, own = (ctypes.c_int32 * n)(), (ctypes.c_int32 * n)()
    sr, sc = (ctypes.c_int64 * n)(), (ctypes.c_int64 * n)()
    sb, rb = (ctypes.c_int64 * world)(), (ctypes.c_int64 * world)()
    ws = ctypes.c_size_t(0)
    rc = _lib().dion2_dist_info(arr, n, ctypes.byref(cfg), world, rank, ax, own, sr, sc, sb, rb, ctypes.byref(ws))
    if rc:
        raise Dion2Error(rc, "dion2_dist_info")
    return {"axis": list(ax), "owner": list(own), "shard": list(zip(sr, sc)), "send_bytes": list(sb),
            "recv_bytes": list(rb), "workspace_bytes": ws.value}


def shard_of(full: torch.Tensor, axis: int, world: int, rank: int) -> torch.Tensor:
    """This rank's shard of a full matrix in the distributed layout: rows mode (axis 0)
    -> column block, cols mode (axis 1) -> row block (contiguous copy)."""
    m, n = full.shape
    if axis == 0:
        b = n // world
        return full[:, rank * b:(rank + 1) * b].contiguous()
    b = m // world
    return full[rank * b:(rank + 1) * b].contiguous()


def _nccl_comm_ptr(group) -> int:
    import torch.distributed as dist
    pg = group if group is not None else dist.group.WORLD
    backend = pg._get_backend(torch.device("cuda"))
    return int(backend._comm_ptr())


class Dion2Dist:
    """Owner-compute distributed Dion2 over a torch.distributed NCCL group (one rank per GPU).

    shapes: the GLOBAL (m, n) of every matrix; each rank passes its local shards
    (see dist_info()["shard"] and shard_of())."""

    def __init__(self, shapes, group=None, m_transposed=None, cuda_graph: bool = False, **cfg_kw):
        """m_transposed: per matrix, the local M shard is stored transposed (column-mode only).
        cuda_graph: a step whose shards and config repeat the previous call's runs eagerly and is
        captured (NCCL calls and the direct-exchange barriers included); later identical steps
        replay the graph, with eta read on the device so a learning-rate schedule still replays.
        Every rank must use the same setting (the captured collectives pair up across ranks)."""
        import torch.distributed as dist
        self.shapes = [tuple(s) for s in shapes]
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cfg_kw = dict(cfg_kw)
        self.m_transposed = m_transposed
        self.cuda_graph = cuda_graph
        self._graph = None
        self._gkey = None
        self._prev_key = None
        self.info = dist_info(self.shapes, self.world, self.rank, m_transposed=m_transposed, **cfg_kw)
        self._ws: Optional[torch.Tensor] = None
        self.last_comm_bytes = 0

    def step(self, Ws, Ms, Gs, sel_out=None, stream=None, **override):
        if self.cuda_graph and stream is None:
            ptrs = lambda ts: tuple((t.data_ptr(), tuple(t.shape), tuple(t.stride()), t.dtype) if t is not None  # noqa: E731
                                    else None for t in ts)
            key = (ptrs(Ws), ptrs(Ms), ptrs(Gs), ptrs(sel_out or ()),
                   tuple(sorted((k, repr(v)) for k, v in {**self.cfg_kw, **override}.items() if k != "lr")),
                   torch.cuda.current_device())
            lr = float({**self.cfg_kw, **override}.get("lr", 0.02))
            if self._graph is not None and key == self._gkey and self._ws is not None:
                self._write_lr(lr)
                self._graph.replay()
                return
            repeat = key == self._prev_key
            self._prev_key = key
            self._step(Ws, Ms, Gs, sel_out, None, lr_device=True, write_lr=lr, **override)
            if repeat:  # the second identical call: capture it (this call's step ran above)
                ws_before = self._ws
                g = torch.cuda.CUDAGraph()
                # thread-local capture: the process group's watchdog thread may query its events
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    self._step(Ws, Ms, Gs, sel_out, None, lr_device=True, **override)
                if self._ws is ws_before:
                    self._graph, self._gkey = g, key
            return
        self._step(Ws, Ms, Gs, sel_out, stream, **override)

    def _write_lr(self, lr: float) -> None:
        """eta into the fp32 word at byte 8 of the 4096-aligned workspace base (stream-ordered)."""
        base = self._ws.data_ptr()
        off = ((base + 4095) & ~4095) - base + 8
        self._ws[off:off + 4].view(torch.float32).fill_(lr)

    def _step(self, Ws, Ms, Gs, sel_out, stream, lr_device: bool = False, write_lr: Optional[float] = None,
              **override):
        kw = dict(self.cfg_kw)
        kw.update(override)
        if lr_device:
            kw["lr_device"] = True
        kw.setdefault("grad_dtype", Gs[0].dtype)
        kw.setdefault("w_dtype", Ws[0].dtype)
        cfg = make_config(**kw)
        dev = Ws[0].device
        need = self.info["workspace_bytes"]
        if self._ws is None or self._ws.numel() < need:
            if self._ws is not None:
                _lib().dion2_release_workspace(self._ws.data_ptr(), self._ws.numel())
            self._ws = torch.empty(need, dtype=torch.uint8, device=dev)
            self._graph = None  # a captured graph references the old workspace
        if write_lr is not None:
            self._write_lr(write_lr)
        arr = _shards(self.shapes, Ws, Ms, Gs, sel_out, self.m_transposed)
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        nbytes = ctypes.c_uint64(0)
        rc = _lib().dion2_step_batched_dist(arr, len(self.shapes), ctypes.byref(cfg), self._ws.data_ptr(),
                                            self._ws.numel(), _nccl_comm_ptr(self.group), self.world, self.rank,
                                            st.cuda_stream, ctypes.byref(nbytes))
        if rc:
            raise Dion2Error(rc, "dion2_step_batched_dist")
        self.last_comm_bytes = nbytes.value

    def status(self):
        bad = ctypes.c_int32(-1)
        rc = _lib().dion2_get_status(self._ws.data_ptr(), torch.cuda.current_stream().cuda_stream, ctypes.byref(bad))
        return rc, bad.value

    def release(self) -> None:
        """Drop the library's plans keyed on this object's workspace (the symmetric windows of a
        direct-exchange plan are tied to its communicator: release before destroying the group)."""
        self._graph = None
        if self._ws is not None:
            _lib().dion2_release_workspace(self._ws.data_ptr(), self._ws.numel())
            self._ws = None

    def __del__(self):
        try:
            self.release()
        except Exception:  # interpreter shutdown: the library may already be gone
            pass

    def exchange_mode(self) -> str:
        """"direct" (peer stores / loads over symmetric memory), "nccl" (send / recv), or
        "none" before the first step."""
        if self._ws is None:
            return "none"
        return {1: "direct", 0: "nccl"}.get(_lib().dion2_dist_exchange_mode(self._ws.data_ptr()), "none")


class Dion2Loopback:
    """All `world` ranks of the distributed step in this process on ONE device; the
    exchanges are device copies (dion2_step_batched_loopback).  For testing the
    distributed layout and kernels without several GPUs."""

    def __init__(self, shapes, world, m_transposed=None, cuda_graph: bool = False, **cfg_kw):
        """cuda_graph: as Dion2Dist (capture on the second identical call, replay after)."""
        self.shapes = [tuple(s) for s in shapes]
        self.world = world
        self.cfg_kw = dict(cfg_kw)
        self.m_transposed = m_transposed
        self.cuda_graph = cuda_graph
        self._graph = None
        self._gkey = None
        self._prev_key = None
        self.infos = [dist_info(self.shapes, world, r, m_transposed=m_transposed, **cfg_kw) for r in range(world)]
        self._ws: List[torch.Tensor] = []
        self.last_comm_bytes = 0

    def step(self, Ws, Ms, Gs, sel_out=None, stream=None, **override):
        """Ws, Ms, Gs: [world][n] local shards; sel_out: optional [world][n] int32 tensors."""
        if self.cuda_graph and stream is None:
            flat = lambda tss: tuple((t.data_ptr(), tuple(t.shape), t.dtype) for ts in tss for t in ts)  # noqa: E731
            key = (flat(Ws), flat(Ms), flat(Gs), flat(sel_out or ()),
                   tuple(sorted((k, repr(v)) for k, v in {**self.cfg_kw, **override}.items())))
            if self._graph is not None and key == self._gkey:
                self._graph.replay()
                return
            repeat = key == self._prev_key
            self._prev_key = key
            self._step(Ws, Ms, Gs, sel_out, None, **override)
            if repeat:
                ws_before = list(self._ws)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    self._step(Ws, Ms, Gs, sel_out, None, **override)
                if self._ws == ws_before:
                    self._graph, self._gkey = g, key
            return
        self._step(Ws, Ms, Gs, sel_out, stream, **override)

    def _step(self, Ws, Ms, Gs, sel_out, stream, **override):
        kw = dict(self.cfg_kw)
        kw.update(override)
        kw.setdefault("grad_dtype", Gs[0][0].dtype)
        kw.setdefault("w_dtype", Ws[0][0].dtype)
        cfg = make_config(**kw)
        n, P = len(self.shapes), self.world
        dev = Ws[0][0].device
        need = max(i["workspace_bytes"] for i in self.infos)
        if len(self._ws) != P or self._ws[0].numel() < need:
            for w in self._ws:
                _lib().dion2_release_workspace(w.data_ptr(), w.numel())
            self._ws = [torch.empty(need, dtype=torch.uint8, device=dev) for _ in range(P)]
            self._graph = None
        arr = (Dion2Shard * (n * P))()
        for r in range(P):
            part = _shards(self.shapes, Ws[r], Ms[r], Gs[r], sel_out[r] if sel_out is not None else None,
                           self.m_transposed)
            for i in range(n):
                arr[r * n + i] = part[i]
        wsp = (ctypes.c_void_p * P)(*[w.data_ptr() for w in self._ws])
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        nbytes = ctypes.c_uint64(0)
        rc = _lib().dion2_step_batched_loopback(arr, n, ctypes.byref(cfg), wsp, need, P, st.cuda_stream,
                                                ctypes.byref(nbytes))
        if rc:
            raise Dion2Error(rc, "dion2_step_batched_loopback")
        self.last_comm_bytes = nbytes.value

    def release(self) -> None:
        """Drop the library's plans keyed on this object's workspaces."""
        self._graph = None
        for w in self._ws:
            _lib().dion2_release_workspace(w.data_ptr(), w.numel())
        self._ws = []

    def __del__(self):
        try:
            self.release()
        except Exception:  # interpreter shutdown: the library may already be gone
            pass


class Dion2DpSync:
    """Compressed DP-sync (paper 3.2): each rank is a data-parallel replica with full W, M
    and its local G; only M[K] is all-reduced (averaged).  Requires select="random"."""

    def __init__(self, group=None, loopback_world: int = 0, m_transposed=None, storage_transposed=None, **cfg_kw):
        """m_transposed: per matrix, M stored transposed (column-mode matrices; every replica
        must use the same flags: the all-reduced buffer holds S^T for those).
        storage_transposed: per matrix, W, M, G held (in, out) (see describe())."""
        cfg_kw.setdefault("select", "random")
        self.cfg_kw = dict(cfg_kw)
        self.m_transposed = m_transposed
        self.storage_transposed = storage_transposed
        self.group = group
        self.loopback = loopback_world > 0
        if self.loopback:
            self.world, self.rank = loopback_world, 0
        else:
            import torch.distributed as dist
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self._ws: List[torch.Tensor] = []
        self.last_comm_bytes = 0

    def _cfg(self, Gs0, override, W0=None):
        kw = dict(self.cfg_kw)
        kw.update(override)
        kw.setdefault("grad_dtype", Gs0.dtype)
        if W0 is not None:
            kw.setdefault("w_dtype", W0.dtype)
        return make_config(**kw)

    def step(self, Ws, Ms, Gs, sel_out=None, stream=None, **override):
        """NCCL mode: this rank's full matrices.  Loopback mode: [world][n] lists."""
        if self.loopback:
            n, P = len(Ws[0]), self.world
            cfg = self._cfg(Gs[0][0], override, Ws[0][0])
            parts = [describe(Ws[r], Ms[r], Gs[r], sel_out[r] if sel_out is not None else None,
                              m_transposed=self.m_transposed, storage_transposed=self.storage_transposed)[0]
                     for r in range(P)]
            arr = (Dion2Matrix * (n * P))()
            for r in range(P):
                for i in range(n):
                    arr[r * n + i] = parts[r][i]
            dev = Ws[0][0].device
        else:
            n, P = len(Ws), self.world
            cfg = self._cfg(Gs[0], override, Ws[0])
            arr, _ = describe(Ws, Ms, Gs, sel_out, m_transposed=self.m_transposed,
                              storage_transposed=self.storage_transposed)
            dev = Ws[0].device
        need = ctypes.c_size_t(0)
        rc = _lib().dion2_dpsync_workspace_size(arr, n, ctypes.byref(cfg), P, ctypes.byref(need))
        if rc:
            raise Dion2Error(rc, "dion2_dpsync_workspace_size")
        nws = P if self.loopback else 1
        if len(self._ws) != nws or self._ws[0].numel() < need.value:
            for w in self._ws:
                _lib().dion2_release_workspace(w.data_ptr(), w.numel())
            self._ws = [torch.empty(need.value, dtype=torch.uint8, device=dev) for _ in range(nws)]
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        nbytes = ctypes.c_uint64(0)
        if self.loopback:
            wsp = (ctypes.c_void_p * P)(*[w.data_ptr() for w in self._ws])
            rc = _lib().dion2_step_batched_dpsync_loopback(arr, n, ctypes.byref(cfg), wsp, need.value, P,
                                                           st.cuda_stream, ctypes.byref(nbytes))
        else:
            rc = _lib().dion2_step_batched_dpsync(arr, n, ctypes.byref(cfg), self._ws[0].data_ptr(), need.value,
                                                  _nccl_comm_ptr(self.group), P, self.rank, st.cuda_stream,
                                                  ctypes.byref(nbytes))
        if rc:
            raise Dion2Error(rc, "dion2_step_batched_dpsync")
        self.last_comm_bytes = nbytes.value

    def release(self) -> None:
        """Drop the library's plans keyed on this object's workspaces (the symmetric windows of a
        direct-exchange plan are tied to its communicator: release before destroying the group)."""
        for w in self._ws:
            _lib().dion2_release_workspace(w.data_ptr(), w.numel())
        self._ws = []

    def __del__(self):
        try:
            self.release()
        except Exception:  # interpreter shutdown: the library may already be gone
            pass

    def exchange_mode(self) -> str:
        """"direct" (peer-memory reduce-scatter / all-gather into symmetric windows) or "nccl"
        (ncclAllReduce), "none" before the first step; loopback reports the mode it emulates."""
        if not self._ws:
            return "none"
        return {1: "direct", 0: "nccl"}.get(_lib().dion2_dist_exchange_mode(self._ws[0].data_ptr()),
                                            "direct" if self.loopback and self.cfg_kw.get("dist_direct") else
                                            ("nccl" if self.loopback else "none"))

    def status(self, replica: int = 0) -> Tuple[int, int]:
        """(code, first bad matrix) of this rank's replica (loopback: of replica `replica`); a
        matrix non-finite on any replica is reported (and skipped) on every replica."""
        bad = ctypes.c_int32(-1)
        rc = _lib().dion2_get_status(self._ws[replica].data_ptr(), torch.cuda.current_stream().cuda_stream,
                                     ctypes.byref(bad))
        return rc, bad.value
