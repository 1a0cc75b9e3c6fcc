"""B200-native data-parallel hot path of arXiv 2110.11226 (stack-based generational GP).

Thin Python binding over the C-ABI in ``include/gp.h`` (``libgp_b200.so``): argument marshalling
only -- every step of evaluation, fitness, reduction and selection runs in the sm_100a kernels,
and mutation runs in the library's C++ host engine. PyTorch supplies device memory, streams and
(for multi-GPU) the process group that broadcasts the NCCL unique id. There is no CPU fallback:
if the extension is missing, loading fails loudly.

Data layout: ``X`` is column-major -- a tensor of shape ``(n_cols, n_rows)`` whose row c
is feature c (``ldx = X.stride(0)``). Programs are a flat CSR: ``nodes`` int32 ``(N, 2)`` (opcode,
var index or float32 bits of the constant) and ``offsets`` int64 ``(n_programs + 1,)``.
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _capi
from ._capi import GpConfig, GpGenerationStats

GP_MAX_STACK = 20
METRICS = {"mae": 0, "mse": 1, "rmse": 2, "logloss": 3, "pearson": 4, "spearman": 5}
HIGHER_IS_BETTER = {"pearson", "spearman"}
OPS = ["var", "const", "add", "sub", "mul", "div", "min", "max", "pow", "sin", "cos", "tan",
       "abs", "neg", "sqrt", "log", "exp", "inv", "square", "cube", "tanh", "sinh", "cosh",
       "asin", "acos", "atan"]
OP = {n: i for i, n in enumerate(OPS)}
FLAGS = {"invalid_prefix": 1, "stack_overflow": 2, "var_range": 4, "nonfinite": 8,
         "undefined_corr": 16, "bad_opcode": 32}
TABLE2_FUNCTIONS = ("add", "sub", "mul", "div", "sin", "cos", "tan")
KIND_NAMES = ["crossover", "subtree", "hoist", "point", "reproduction"]


class GPError(RuntimeError):
    pass


def lib():
    return _capi.lib()


def _check(status: int, ctx_handle=None, what: str = ""):
    if status != 0:
        L = lib()
        name = L.gp_status_string(status).decode()
        msg = (L.gp_last_error(ctx_handle) or b"").decode()
        raise GPError(f"{what}: {name}: {msg}")


def _ptr(t):
    """Raw pointer of a torch tensor (host or device) or numpy array; None -> NULL."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _metric_id(metric) -> int:
    return METRICS[metric] if isinstance(metric, str) else int(metric)


def get_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it and broadcasts it to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().gp_get_unique_id(buf), None, "gp_get_unique_id")
    return buf.raw


def config(**kw) -> GpConfig:
    """gp_config with Table 6 defaults (gp_config_default) and keyword overrides. ``metric`` and
    ``function_set`` accept names."""
    c = GpConfig()
    lib().gp_config_default(ctypes.byref(c))
    for k, v in kw.items():
        if k == "metric":
            v = _metric_id(v)
        if k == "function_set":
            ops = [OP[f] if isinstance(f, str) else int(f) for f in v]
            c.n_functions = len(ops)
            for i, o in enumerate(ops):
                c.function_set[i] = o
            continue
        if not hasattr(c, k):
            raise KeyError(f"unknown gp_config field {k!r}")
        setattr(c, k, v)
    return c


class Context:
    """gp_context: device, stream and (optionally) an NCCL communicator over the ranks."""

    def __init__(self, device: int = 0, stream=None, unique_id: bytes | None = None,
                 rank: int = 0, world_size: int = 1):
        import torch
        torch.cuda.set_device(device)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.device, self.rank, self.world_size = device, rank, world_size
        self.stream = stream
        h = ctypes.c_void_p()
        uid = None if unique_id is None else ctypes.create_string_buffer(unique_id, 128)
        _check(lib().gp_context_create(ctypes.byref(h), device, ctypes.c_void_p(stream.cuda_stream),
                                       uid, rank, world_size), None, "gp_context_create")
        self.handle = h
        self._engines = weakref.WeakSet()      # engines on this context (closed first)

    def close(self):
        if getattr(self, "handle", None):
            for e in list(getattr(self, "_engines", ())):
                e.close()
            lib().gp_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, enabled: bool = True):
        _check(lib().gp_context_set_profiling(self.handle, int(enabled)), self.handle, "profiling")

    def eval_timing(self, reset: bool = True):
        """(total eval-kernel ms, launches) recorded with CUDA events on the context stream."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(lib().gp_context_eval_timing(self.handle, ctypes.byref(ms), ctypes.byref(n),
                                            int(reset)), self.handle, "eval_timing")
        return ms.value, n.value

    def set_shard(self, mode: str = "rows"):
        """gp_context_set_shard: "rows" (each rank passes its row shard; partial sums all-reduced)
        or "programs" (each rank passes all rows, evaluates its program chunk; fitness
        all-gathered)."""
        _check(lib().gp_context_set_shard(self.handle, {"rows": 0, "programs": 1}[mode]),
               self.handle, "set_shard")

    def set_const_programs(self, closed_form: bool = True):
        """gp_context_set_const_programs: variable-free programs' MSE / RMSE / Pearson fitness from
        the dataset moments (default) or through the per-row evaluator."""
        _check(lib().gp_context_set_const_programs(self.handle, int(bool(closed_form))), self.handle,
               "set_const_programs")

    def set_eval_order(self, sethi_ullman: bool = True):
        """Sethi-Ullman operand order (default) or the classic reverse-prefix order."""
        _check(lib().gp_context_set_eval_order(self.handle, int(bool(sethi_ullman))), self.handle,
               "set_eval_order")

    def kernel_launches(self, reset: bool = True) -> int:
        """CUDA kernels launched by the library on this context since the last reset."""
        n = ctypes.c_int64()
        _check(lib().gp_context_kernel_launches(self.handle, ctypes.byref(n), int(reset)),
               self.handle, "kernel_launches")
        return n.value

    def set_reference_row(self, x_row, y_ref: float):
        x = np.ascontiguousarray(np.asarray(x_row, np.float32))
        _check(lib().gp_context_set_reference_row(self.handle, x.ctypes.data, len(x),
                                                  float(y_ref)), self.handle, "reference row")

    def evaluate(self, nodes, offsets, X, y, w=None, metric="mse", max_stack: int = GP_MAX_STACK,
                 fitness_out=None, status_out=None, n_rows: int | None = None):
        """gp_evaluate. Returns (fitness float32 [n], status uint32-as-int32 [n]) on X's device
        (or the given output tensors)."""
        import torch
        n = offsets.shape[0] - 1
        n_rows = X.shape[1] if n_rows is None else n_rows
        dev = X.device if isinstance(X, torch.Tensor) else torch.device("cpu")
        if fitness_out is None:
            fitness_out = torch.empty(n, dtype=torch.float32, device=dev)
        if status_out is None:
            status_out = torch.empty(n, dtype=torch.int32, device=dev)
        _check(lib().gp_evaluate(self.handle, _ptr(nodes), _ptr(offsets), n, int(nodes.shape[0]),
                                 int(max_stack), _ptr(X), int(X.stride(0) if isinstance(X, torch.Tensor)
                                                              else X.strides[0] // 4),
                                 _ptr(y), _ptr(w), int(n_rows), int(X.shape[0]), _metric_id(metric),
                                 _ptr(fitness_out), _ptr(status_out)), self.handle, "gp_evaluate")
        return fitness_out, status_out

    def evaluate_partial(self, nodes, offsets, X, y, w=None, metric="mse",
                         max_stack: int = GP_MAX_STACK, sums_out=None, n_rows: int | None = None):
        """gp_evaluate_partial: fp64 per-program sums of these rows (program order, S per
        program, then W, S_y, S_yy). Returns sums_out (float64 on X's device by default)."""
        import torch
        n = offsets.shape[0] - 1
        S = 3 if metric == "pearson" else 1
        n_rows = X.shape[1] if n_rows is None else n_rows
        if sums_out is None:
            sums_out = torch.empty(n * S + 3, dtype=torch.float64, device=X.device)
        _check(lib().gp_evaluate_partial(self.handle, _ptr(nodes), _ptr(offsets), n,
                                         int(nodes.shape[0]), int(max_stack), _ptr(X),
                                         int(X.stride(0)), _ptr(y), _ptr(w), int(n_rows),
                                         int(X.shape[0]), _metric_id(metric), _ptr(sums_out)),
               self.handle, "gp_evaluate_partial")
        return sums_out

    def finalize_sums(self, nodes, offsets, sums, n_cols: int, metric="mse",
                      max_stack: int = GP_MAX_STACK, fitness_out=None, status_out=None):
        """gp_finalize_sums: fitness / status from (shard-summed) gp_evaluate_partial sums."""
        import torch
        n = offsets.shape[0] - 1
        dev = sums.device
        if fitness_out is None:
            fitness_out = torch.empty(n, dtype=torch.float32, device=dev)
        if status_out is None:
            status_out = torch.empty(n, dtype=torch.int32, device=dev)
        _check(lib().gp_finalize_sums(self.handle, _ptr(nodes), _ptr(offsets), n,
                                      int(nodes.shape[0]), int(max_stack), int(n_cols), _ptr(sums),
                                      _metric_id(metric), _ptr(fitness_out), _ptr(status_out)),
               self.handle, "gp_finalize_sums")
        return fitness_out, status_out

    def set_plan(self, group_size: int = 0, tiles_per_chunk: int = 0):
        """gp_context_set_plan (0 = automatic)."""
        _check(lib().gp_context_set_plan(self.handle, int(group_size), int(tiles_per_chunk)),
               self.handle, "gp_context_set_plan")

    def set_program_range(self, lo: int = 0, hi: int = -1):
        """gp_context_set_program_range ([lo, hi); hi < 0 = all)."""
        _check(lib().gp_context_set_program_range(self.handle, int(lo), int(hi)), self.handle,
               "gp_context_set_program_range")

    def predict(self, nodes, offsets, X, max_stack: int = GP_MAX_STACK, out=None, status_out=None):
        """gp_predict: out[p, i] = f_p(x_i) (float32, device)."""
        import torch
        n = offsets.shape[0] - 1
        n_rows = X.shape[1]
        if out is None:
            out = torch.full((n, n_rows), float("nan"), dtype=torch.float32, device=X.device)
        if status_out is None:
            status_out = torch.empty(n, dtype=torch.int32, device=X.device)
        _check(lib().gp_predict(self.handle, _ptr(nodes), _ptr(offsets), n, int(nodes.shape[0]),
                                int(max_stack), _ptr(X), int(X.stride(0)), int(n_rows),
                                int(X.shape[0]), _ptr(out), int(out.stride(0)), _ptr(status_out)),
               self.handle, "gp_predict")
        return out, status_out

    def tournament_select(self, fitness, offsets, n_tournaments: int, tournament_size: int = 4,
                          parsimony: float = 0.01, higher_is_better: bool = False, seed: int = 2110,
                          generation: int = 0, winners_out=None):
        import torch
        n = offsets.shape[0] - 1
        if winners_out is None:
            winners_out = torch.empty(n_tournaments, dtype=torch.int32, device=fitness.device)
        _check(lib().gp_tournament_select(self.handle, _ptr(fitness), _ptr(offsets), n,
                                          n_tournaments, tournament_size, float(parsimony),
                                          int(bool(higher_is_better)), int(seed), int(generation),
                                          _ptr(winners_out)), self.handle, "gp_tournament_select")
        return winners_out


class Engine:
    """gp_engine: Alg. 1 -- GPU selection + evaluation, host C++ mutation."""

    def __init__(self, ctx: Context, X, y, w=None, cfg: GpConfig | None = None, **kw):
        self.ctx = ctx
        self.cfg = cfg if cfg is not None else config(**kw)
        self._keep = (X, y, w)
        h = ctypes.c_void_p()
        _check(lib().gp_engine_create(ctypes.byref(h), ctx.handle, ctypes.byref(self.cfg), _ptr(X),
                                      int(X.stride(0)), _ptr(y), _ptr(w), int(X.shape[1]),
                                      int(X.shape[0])), ctx.handle, "gp_engine_create")
        self.handle = h
        ctx._engines.add(self)

    def set_dataset(self, X, y, w=None):
        self._keep = (X, y, w)
        _check(lib().gp_engine_set_dataset(self.handle, _ptr(X), int(X.stride(0)), _ptr(y), _ptr(w),
                                           int(X.shape[1]), int(X.shape[0])),
               self.ctx.handle, "gp_engine_set_dataset")

    def init_population(self) -> dict:
        st = GpGenerationStats()
        _check(lib().gp_engine_init_population(self.handle, ctypes.byref(st)), self.ctx.handle,
               "gp_engine_init_population")
        return st.as_dict()

    def generation(self) -> dict:
        st = GpGenerationStats()
        _check(lib().gp_generation(self.handle, ctypes.byref(st)), self.ctx.handle, "gp_generation")
        return st.as_dict()

    def population(self):
        """Copies of the current population: (nodes (N,2) int32, offsets int64, fitness f32)."""
        nodes, off, fit = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        n, nn = ctypes.c_int32(), ctypes.c_int64()
        _check(lib().gp_engine_population(self.handle, ctypes.byref(nodes), ctypes.byref(off),
                                          ctypes.byref(fit), ctypes.byref(n), ctypes.byref(nn)),
               self.ctx.handle, "gp_engine_population")
        N = nn.value
        nodes_np = np.ctypeslib.as_array(ctypes.cast(nodes, ctypes.POINTER(ctypes.c_int32)),
                                         (N * 2,)).reshape(N, 2).copy()
        off_np = np.ctypeslib.as_array(ctypes.cast(off, ctypes.POINTER(ctypes.c_int64)),
                                       (n.value + 1,)).copy()
        fit_np = np.ctypeslib.as_array(ctypes.cast(fit, ctypes.POINTER(ctypes.c_float)),
                                       (n.value,)).copy()
        return nodes_np, off_np, fit_np

    def population_device(self):
        """Device copies (torch, cuda) of the current population: (nodes (N,2) int32, offsets
        int64, fitness f32) -- gp_engine_population_device views, cloned."""
        import torch
        nodes, off, fit = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        n, nn = ctypes.c_int32(), ctypes.c_int64()
        _check(lib().gp_engine_population_device(self.handle, ctypes.byref(nodes),
                                                 ctypes.byref(off), ctypes.byref(fit),
                                                 ctypes.byref(n), ctypes.byref(nn)),
               self.ctx.handle, "gp_engine_population_device")
        dev = torch.device("cuda", self.ctx.device)
        out_n = torch.empty((nn.value, 2), dtype=torch.int32, device=dev)
        out_o = torch.empty(n.value + 1, dtype=torch.int64, device=dev)
        out_f = torch.empty(n.value, dtype=torch.float32, device=dev)
        torch.cuda.synchronize(dev)
        for dst, src in ((out_n, nodes), (out_o, off), (out_f, fit)):
            _check(lib().gp_device_copy(_ptr(dst), src, dst.numel() * dst.element_size()),
                   self.ctx.handle, "copy")
        return out_n, out_o, out_f

    def set_population(self, nodes, offsets, fitness=None, generation: int = 0,
                       stats: bool = True):
        """gp_engine_set_population ([host|device] flat CSR; fitness None = evaluate now).
        stats=False skips the statistics (no synchronisation for device inputs); returns the
        statistics dict or None."""
        self._keep_pop = (nodes, offsets, fitness)
        st = GpGenerationStats()
        _check(lib().gp_engine_set_population(self.handle, _ptr(nodes), _ptr(offsets),
                                              int(offsets.shape[0] - 1), int(nodes.shape[0]),
                                              _ptr(fitness), int(generation),
                                              ctypes.byref(st) if stats else None),
               self.ctx.handle, "gp_engine_set_population")
        return st.as_dict() if stats else None

    def last_selection(self):
        """(kinds int32 [n], winners int32 [T]) of the last gp_generation."""
        k, w = ctypes.c_void_p(), ctypes.c_void_p()
        t = ctypes.c_int32()
        _check(lib().gp_engine_last_selection(self.handle, ctypes.byref(k), ctypes.byref(w),
                                              ctypes.byref(t)), self.ctx.handle, "last_selection")
        n = self.cfg.population_size
        if not k.value or not w.value:
            return np.zeros(0, np.int32), np.zeros(0, np.int32)
        kinds = np.ctypeslib.as_array(ctypes.cast(k, ctypes.POINTER(ctypes.c_int32)), (n,)).copy()
        winners = np.ctypeslib.as_array(ctypes.cast(w, ctypes.POINTER(ctypes.c_int32)),
                                        (t.value,)).copy()
        return kinds, winners

    def close(self):
        if getattr(self, "handle", None) and getattr(self.ctx, "handle", None):
            lib().gp_engine_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
