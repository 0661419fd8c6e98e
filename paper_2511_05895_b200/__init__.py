"""paper_2511_05895_b200 -- B200-native dynamic max-flow (arXiv 2511.05895).

Thin Python binding over the C ABI of ``libdmf.so`` (include/dmf.h).  This module
only marshals arguments: every step of the hot path (batch validation and
Updates Processing, global-relabel BFS, worklist compaction, push / pull
discharge, RemoveInvalidEdges, push-pull stages, flow value, cuts) runs in the
library's sm_100a kernels.  There is no CPU fallback: if the extension is missing
or no CUDA device is present the constructor raises.

PyTorch is used for device memory (optional caching-allocator hook) and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB as _LIB_PATH

__all__ = ["DynMaxFlow", "DMFError", "load_library", "DYN_PR", "DYN_PP", "CAP_MAX", "STATUS"]

DYN_PR, DYN_PP = 0, 1
CAP_MAX = 1073741823
STATUS = {0: "DMF_OK", -1: "DMF_EINVAL", -2: "DMF_ENOSLOT", -3: "DMF_EDUP", -4: "DMF_ESTATE",
          -5: "DMF_ENOMEM", -6: "DMF_ECUDA", -7: "DMF_EOVERFLOW", -8: "DMF_ENOCONV", -9: "DMF_ECHECK"}
SCHED = {"auto": 0, "async": 1, "rounds": 2, "topology": 3}
_ALGO = {"pr": DYN_PR, "pp": DYN_PP, DYN_PR: DYN_PR, DYN_PP: DYN_PP}

_ALLOC_T = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_FREE_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)


class Options(ctypes.Structure):
    """dmf_options (include/dmf.h): field order and types mirror the C struct."""
    _fields_ = [("kernel_cycles", ctypes.c_int32), ("algo", ctypes.c_int32), ("max_iters", ctypes.c_int32),
                ("grid_blocks", ctypes.c_int32), ("stream", ctypes.c_void_p), ("alloc", _ALLOC_T),
                ("free", _FREE_T), ("alloc_ctx", ctypes.c_void_p),
                ("schedule", ctypes.c_int32), ("async_warps", ctypes.c_int32), ("budget_mul", ctypes.c_int32),
                ("tail_items", ctypes.c_int32), ("local_gap", ctypes.c_int32), ("warm", ctypes.c_int32),
                ("topo_div", ctypes.c_int32), ("check_level", ctypes.c_int32), ("certify", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 7)]


KNOBS = ("schedule", "async_warps", "budget_mul", "tail_items", "local_gap", "warm", "topo_div", "check_level",
         "certify")


class Stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("S", ctypes.c_int64),
                ("kernel_cycles", ctypes.c_int32), ("grid_blocks", ctypes.c_int32), ("block_threads", ctypes.c_int32),
                ("iterations", ctypes.c_int64), ("bfs_levels", ctypes.c_int64), ("bfs_vertices", ctypes.c_int64),
                ("bfs_slots", ctypes.c_int64), ("discharge_vertices", ctypes.c_int64),
                ("discharge_slots", ctypes.c_int64), ("pushes", ctypes.c_int64), ("relabels", ctypes.c_int64),
                ("rie_slots", ctypes.c_int64), ("rie_saturations", ctypes.c_int64),
                ("batch_entries", ctypes.c_int64), ("stage2_vertices", ctypes.c_int64),
                ("stage2_iterations", ctypes.c_int64), ("rounds", ctypes.c_int64), ("activations", ctypes.c_int64),
                ("reset_vertices", ctypes.c_int64), ("budget_stops", ctypes.c_int64), ("bottom_up_levels", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64),
                ("device_ms", ctypes.c_float), ("t_prologue_us", ctypes.c_float), ("t_reset_us", ctypes.c_float),
                ("t_bfs_us", ctypes.c_float), ("t_discharge_us", ctypes.c_float), ("t_rie_us", ctypes.c_float),
                ("t_epilogue_us", ctypes.c_float), ("gap_levels", ctypes.c_int64), ("gap_skips", ctypes.c_int64),
                ("topology_rounds", ctypes.c_int64), ("tail_stops", ctypes.c_int64), ("stage2_skipped", ctypes.c_int64),
                ("certified", ctypes.c_int64), ("query_ms", ctypes.c_float),
                ("query_bfs_vertices", ctypes.c_int64), ("query_bfs_slots", ctypes.c_int64)]


class DMFError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


_lib = None


def load_library():
    """Load libdmf.so (built in-tree by build.py / __graft_entry__.build()).  Fails
    loudly if it is missing: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"libdmf.so not built ({_LIB_PATH}); run python -m paper_2511_05895_b200.build")
        L = ctypes.CDLL(_LIB_PATH)
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.dmf_default_options.argtypes = [ctypes.POINTER(Options)]
        L.dmf_default_options.restype = None
        L.dmf_create.argtypes = [I32, P, P, P, I32, I32, ctypes.POINTER(Options), ctypes.POINTER(P)]
        L.dmf_static_solve.argtypes = [P]
        L.dmf_apply_batch.argtypes = [P, I64, P, P, P, I32]
        L.dmf_flow_value.argtypes = [P, ctypes.POINTER(I64)]
        L.dmf_min_cut_source_side.argtypes = [P, P]
        L.dmf_max_cut_source_side.argtypes = [P, P]
        L.dmf_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
        L.dmf_sizes.argtypes = [P, ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.dmf_export_state.argtypes = [P, P, P, P, P, P, P]
        L.dmf_export_labels.argtypes = [P, P, P, P, P]
        L.dmf_to_flow.argtypes = [P]
        L.dmf_import_state.argtypes = [P, P, P, P]
        L.dmf_check_state.argtypes = [P]
        L.dmf_static_solve_pp.argtypes = [P]
        L.dmf_edge_flow.argtypes = [P, P]
        L.dmf_set_trace.argtypes = [P, I32]
        L.dmf_get_trace.argtypes = [P, P, I32, ctypes.POINTER(I32)]
        L.dmf_get_trace_cta.argtypes = [P, P, I32, ctypes.POINTER(I32)]
        L.dmf_destroy.argtypes = [P]
        L.dmf_destroy.restype = None
        L.dmf_last_error.restype = ctypes.c_char_p
        for f in ("dmf_create", "dmf_static_solve", "dmf_static_solve_pp", "dmf_apply_batch", "dmf_flow_value", "dmf_min_cut_source_side",
                  "dmf_max_cut_source_side", "dmf_get_stats", "dmf_sizes", "dmf_export_state", "dmf_export_labels", "dmf_to_flow", "dmf_edge_flow", "dmf_set_trace",
                  "dmf_import_state", "dmf_check_state",
                  "dmf_get_trace", "dmf_get_trace_cta"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    """Pointer of a numpy array (host) or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(a.data_ptr())


def _i32(a, name="array"):
    """int32, contiguous, 1-D: numpy arrays are converted, torch tensors must already be."""
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, np.int32)
    else:
        import torch
        if not isinstance(a, torch.Tensor):
            a = np.ascontiguousarray(np.asarray(a), np.int32)
        elif a.dtype != torch.int32 or not a.is_contiguous():
            raise TypeError(f"{name}: torch tensors must be contiguous int32 (got {a.dtype}, contiguous={a.is_contiguous()})")
    if a.ndim != 1:
        raise ValueError(f"{name}: expected a 1-D array, got shape {tuple(a.shape)}")
    return a


class DynMaxFlow:
    """One max-flow instance on one GPU (dmf_graph handle).

    >>> f = DynMaxFlow(n, row_ptr, col, cap, s, t)      # dmf_create
    >>> F = f.static_solve()                              # dmf_static_solve
    >>> F = f.apply_batch(u, v, new_cap, algo="pp")       # dmf_apply_batch
    >>> mask = f.min_cut_source_side()                    # dmf_min_cut_source_side
    """

    def __init__(self, n, row_ptr, col, cap, s, t, kernel_cycles=0, algo="pp", max_iters=0, grid_blocks=0,
                 torch_alloc=True, stream=None, **knobs):
        L = load_library()
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("DynMaxFlow needs a CUDA device (B200); there is no CPU path")
        self._L = L
        self._torch = torch
        opt = Options()
        L.dmf_default_options(ctypes.byref(opt))
        opt.kernel_cycles = kernel_cycles
        opt.algo = _ALGO[algo]
        opt.max_iters = max_iters
        opt.grid_blocks = grid_blocks
        for k, val in knobs.items():          # per-handle engine knobs (dmf_options; include/dmf.h)
            if k not in KNOBS:
                raise TypeError(f"unknown option {k!r} (expected one of {KNOBS})")
            setattr(opt, k, SCHED[val] if k == "schedule" and isinstance(val, str) else int(val))
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        # torch's default stream has handle 0, which the library would read as "create
        # my own stream": pass cudaStreamLegacy instead so that library work stays
        # ordered with torch work on the default stream
        opt.stream = ctypes.c_void_p(stream.cuda_stream if stream.cuda_stream else 1)
        self._cbs = None
        if torch_alloc:
            dev = torch.cuda.current_device()
            _cal, _cdel = torch.cuda.caching_allocator_alloc, torch.cuda.caching_allocator_delete

            def _alloc(nbytes, ctx):
                try:
                    return _cal(int(nbytes), dev, stream)
                except Exception:
                    return None

            def _free(p, nbytes, ctx):
                try:
                    _cdel(int(p))
                except Exception:
                    pass

            self._cbs = (_ALLOC_T(_alloc), _FREE_T(_free))
            opt.alloc, opt.free = self._cbs
        rp = np.ascontiguousarray(row_ptr, np.int64) if isinstance(row_ptr, np.ndarray) else row_ptr
        col = _i32(col, "col")
        cap = _i32(cap, "cap")
        if col.shape[0] != cap.shape[0]:
            raise ValueError(f"col and cap differ in length ({col.shape[0]} vs {cap.shape[0]})")
        h = ctypes.c_void_p()
        rc = L.dmf_create(int(n), _ptr(rp), _ptr(col), _ptr(cap), int(s), int(t), ctypes.byref(opt), ctypes.byref(h))
        self._check(rc)
        self._h = h
        self.n, self.s, self.t = int(n), int(s), int(t)
        n32, S, m = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        L.dmf_sizes(h, ctypes.byref(n32), ctypes.byref(S), ctypes.byref(m))
        self.S, self.m = S.value, m.value

    @classmethod
    def from_graph(cls, g, **kw):
        """Build from a workloads.Graph-like edge list (n, s, t, u, v, cap)."""
        order = np.argsort(g.u, kind="stable")
        counts = np.bincount(g.u, minlength=g.n).astype(np.int64)
        row_ptr = np.zeros(g.n + 1, np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        return cls(g.n, row_ptr, np.ascontiguousarray(g.v[order], np.int32),
                   np.ascontiguousarray(g.cap[order], np.int32), g.s, g.t, **kw)

    def _check(self, rc):
        if rc != 0:
            raise DMFError(rc, self._L.dmf_last_error().decode())

    def static_solve(self) -> int:
        self._check(self._L.dmf_static_solve(self._h))
        return self.flow_value()

    def static_solve_pp(self) -> int:
        """Static push-pull solve: t's in-edges saturated too; returns F."""
        self._check(self._L.dmf_static_solve_pp(self._h))
        return self.flow_value()

    def apply_batch(self, u, v, new_cap, algo=None) -> int:
        u, v, c = _i32(u, "u"), _i32(v, "v"), _i32(new_cap, "new_cap")
        k = int(u.shape[0])
        if v.shape[0] != k or c.shape[0] != k:
            raise ValueError(f"u, v, new_cap must have equal lengths (got {k}, {v.shape[0]}, {c.shape[0]})")
        a = -1 if algo is None else _ALGO[algo]
        self._check(self._L.dmf_apply_batch(self._h, k, _ptr(u), _ptr(v), _ptr(c), a))
        return self.flow_value()

    def flow_value(self) -> int:
        out = ctypes.c_int64()
        self._check(self._L.dmf_flow_value(self._h, ctypes.byref(out)))
        return out.value

    def min_cut_source_side(self, out=None):
        if out is None:
            out = np.zeros(self.n, np.uint8)
        self._check(self._L.dmf_min_cut_source_side(self._h, _ptr(out)))
        return out

    def max_cut_source_side(self, out=None):
        if out is None:
            out = np.zeros(self.n, np.uint8)
        self._check(self._L.dmf_max_cut_source_side(self._h, _ptr(out)))
        return out

    def stats(self) -> dict:
        return self.stats_to_dict(self.raw_stats())

    def raw_stats(self, into: "Stats | None" = None) -> Stats:
        """dmf_get_stats into a ctypes struct (cheap; convert later with stats_to_dict)."""
        st = into if into is not None else Stats()
        self._check(self._L.dmf_get_stats(self._h, ctypes.byref(st)))
        return st

    @staticmethod
    def stats_to_dict(st: Stats) -> dict:
        return {f: getattr(st, f) for f, _ in Stats._fields_}

    PHASES = {0: "prologue", 1: "reset", 2: "bfs", 3: "discharge", 4: "rie", 5: "epilogue", 6: "bfs_bu", 7: "bfs_cmp"}

    def set_trace(self, capacity: int = 4096):
        self._check(self._L.dmf_set_trace(self._h, int(capacity)))

    def trace(self) -> list:
        """Per-phase records of the last call: dicts (phase, iter, sub, items, extra, us)."""
        cnt = ctypes.c_int32()
        self._check(self._L.dmf_get_trace(self._h, None, 0, ctypes.byref(cnt)))
        buf = np.zeros(8 * max(cnt.value, 1), np.int32)
        self._check(self._L.dmf_get_trace(self._h, _ptr(buf), cnt.value, ctypes.byref(cnt)))
        out = []
        for r in buf[:8 * cnt.value].reshape(-1, 8):
            out.append(dict(phase=self.PHASES.get(int(r[0]), int(r[0])), iter=int(r[1]), sub=int(r[2]),
                            items=int(r[3]), extra=int(r[4]), us=float(r[5]) * 1e-3,
                            slow_us=float(np.uint32(r[6])) * 1e-3, slow_deg=int(np.uint32(r[7])) >> 8,
                            slow_cyc=int(np.uint32(r[7])) & 255))
        return out

    def trace_cta(self) -> np.ndarray:
        """Per-CTA busy time (us) of every trace record of the last call: [records, grid]."""
        cnt = ctypes.c_int32()
        self._check(self._L.dmf_get_trace(self._h, None, 0, ctypes.byref(cnt)))
        grid = ctypes.c_int32()
        self._check(self._L.dmf_get_trace_cta(self._h, None, 0, ctypes.byref(grid)))
        buf = np.zeros(max(cnt.value, 1) * grid.value, np.uint32)
        self._check(self._L.dmf_get_trace_cta(self._h, _ptr(buf), cnt.value, ctypes.byref(grid)))
        return buf[:cnt.value * grid.value].reshape(cnt.value, grid.value).astype(np.float64) * 1e-3

    def export_state(self) -> dict:
        row_ptr = np.zeros(self.n + 1, np.int64)
        dst = np.zeros(self.S, np.int32)
        rev = np.zeros(self.S, np.int32)
        cap = np.zeros(self.S, np.int32)
        res = np.zeros(self.S, np.int32)
        e = np.zeros(self.n, np.int64)
        self._check(self._L.dmf_export_state(self._h, _ptr(row_ptr), _ptr(dst), _ptr(rev), _ptr(cap), _ptr(res), _ptr(e)))
        return dict(row_ptr=row_ptr, dst=dst, rev=rev, cap=cap, res=res, e=e)

    def import_state(self, cap, res, excess):
        """dmf_import_state: restore (cap, res, excess) exported from a handle of the same
        input graph; the state is then valid but not converged (repair with a DYN_PR batch)."""
        cap, res = _i32(cap, "cap"), _i32(res, "res")
        e = np.ascontiguousarray(excess, np.int64) if isinstance(excess, np.ndarray) else excess
        if cap.shape[0] != self.S or res.shape[0] != self.S or e.shape[0] != self.n:
            raise ValueError("import_state: cap/res need S entries and excess n entries")
        self._check(self._L.dmf_import_state(self._h, _ptr(cap), _ptr(res), _ptr(e)))

    def check_state(self):
        """dmf_check_state: device invariant check of the current state (raises DMFError)."""
        self._check(self._L.dmf_check_state(self._h))

    def to_flow(self) -> int:
        """Stage (ii): convert the state into a true maximum flow (dmf_to_flow); returns F."""
        self._check(self._L.dmf_to_flow(self._h))
        return self.flow_value()

    def edge_flow(self, out=None):
        """Per-slot flow max(0, cap - res), int32[S] in dmf_export_state's slot order."""
        out = np.zeros(self.S, np.int32) if out is None else out
        self._check(self._L.dmf_edge_flow(self._h, _ptr(out)))
        return out

    def export_labels(self) -> dict:
        hp = np.zeros(self.n, np.int32)
        hm = np.zeros(self.n, np.int32)
        part = np.zeros(self.n, np.uint8)
        rres = np.zeros(self.S, np.int32)
        self._check(self._L.dmf_export_labels(self._h, _ptr(hp), _ptr(hm), _ptr(part), _ptr(rres)))
        return dict(hp=hp, hm=hm, part=part, rres=rres)

    def close(self):
        if getattr(self, "_h", None):
            self._L.dmf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
