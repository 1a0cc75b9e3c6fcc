"""ctypes declarations of include/gp.h (argument marshalling only; no compute here)."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# GP_B200_LIB overrides the library path (experiments: alternative kernel shapes)
LIB_PATH = os.environ.get("GP_B200_LIB", os.path.join(HERE, "libgp_b200.so"))

P = ctypes.c_void_p
i32, i64, u32, u64, f32, f64 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64,
                                ctypes.c_float, ctypes.c_double)

# Entry points and their (argtypes, restype); the CPU test checks each is exported.
SIGNATURES = {
    "gp_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "gp_last_error": ([P], ctypes.c_char_p),
    "gp_version": ([], ctypes.c_char_p),
    "gp_get_unique_id": ([P], ctypes.c_int),
    "gp_context_create": ([ctypes.POINTER(P), ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int],
                          ctypes.c_int),
    "gp_context_destroy": ([P], ctypes.c_int),
    "gp_context_set_stream": ([P, P], ctypes.c_int),
    "gp_context_set_reference_row": ([P, P, i32, f32], ctypes.c_int),
    "gp_context_set_profiling": ([P, ctypes.c_int], ctypes.c_int),
    "gp_context_eval_timing": ([P, ctypes.POINTER(f64), ctypes.POINTER(i64), ctypes.c_int],
                               ctypes.c_int),
    "gp_context_kernel_launches": ([P, ctypes.POINTER(i64), ctypes.c_int], ctypes.c_int),
    "gp_context_set_eval_order": ([P, ctypes.c_int], ctypes.c_int),
    "gp_context_set_const_programs": ([P, ctypes.c_int], ctypes.c_int),
    "gp_context_set_shard": ([P, ctypes.c_int], ctypes.c_int),
    "gp_evaluate": ([P, P, P, i32, i64, i32, P, i64, P, P, i64, i32, ctypes.c_int, P, P],
                    ctypes.c_int),
    "gp_evaluate_partial": ([P, P, P, i32, i64, i32, P, i64, P, P, i64, i32, ctypes.c_int, P],
                            ctypes.c_int),
    "gp_finalize_sums": ([P, P, P, i32, i64, i32, i32, P, ctypes.c_int, P, P], ctypes.c_int),
    "gp_context_set_plan": ([P, i32, i64], ctypes.c_int),
    "gp_context_set_program_range": ([P, i32, i32], ctypes.c_int),
    "gp_predict": ([P, P, P, i32, i64, i32, P, i64, i64, i32, P, i64, P], ctypes.c_int),
    "gp_tournament_select": ([P, P, P, i32, i32, i32, f32, i32, u64, u32, P], ctypes.c_int),
    "gp_config_default": ([P], None),
    "gp_engine_create": ([ctypes.POINTER(P), P, P, P, i64, P, P, i64, i32], ctypes.c_int),
    "gp_engine_set_dataset": ([P, P, i64, P, P, i64, i32], ctypes.c_int),
    "gp_engine_destroy": ([P], ctypes.c_int),
    "gp_engine_init_population": ([P, P], ctypes.c_int),
    "gp_generation": ([P, P], ctypes.c_int),
    "gp_engine_population": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                              ctypes.POINTER(i32), ctypes.POINTER(i64)], ctypes.c_int),
    "gp_engine_population_device": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                     ctypes.POINTER(i32), ctypes.POINTER(i64)], ctypes.c_int),
    "gp_engine_set_population": ([P, P, P, i32, i64, P, i32, P], ctypes.c_int),
    "gp_device_copy": ([P, P, ctypes.c_size_t], ctypes.c_int),
    "gp_engine_last_selection": ([P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(i32)],
                                 ctypes.c_int),
}


class GpConfig(ctypes.Structure):
    """gp_config (include/gp.h)."""
    _fields_ = [
        ("population_size", i32), ("tournament_size", i32), ("parsimony", f32), ("metric", i32),
        ("p_crossover", f64), ("p_subtree", f64), ("p_hoist", f64), ("p_point", f64),
        ("p_point_replace", f64), ("init_depth_min", i32), ("init_depth_max", i32),
        ("const_lo", f32), ("const_hi", f32), ("n_functions", i32), ("function_set", i32 * 32),
        ("stack_capacity", i32), ("seed", u64), ("n_threads", i32), ("device_mutation", i32),
    ]


class GpGenerationStats(ctypes.Structure):
    """gp_generation_stats (include/gp.h)."""
    _fields_ = [
        ("generation", i32), ("best_raw", f32), ("best_adjusted", f32), ("best_index", i32),
        ("best_len", i32), ("best_depth", i32), ("mean_raw", f64), ("total_nodes", i64),
        ("max_stack_need", i32), ("n_tournaments", i32), ("t_select_s", f64),
        ("t_mutate_s", f64), ("t_h2d_s", f64), ("t_eval_s", f64), ("t_total_s", f64),
        ("op_count", i64 * 26), ("const_nodes", i64), ("const_programs", i64),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["op_count"] = list(self.op_count)
        return d


_lib = None


def lib() -> ctypes.CDLL:
    """Loads libgp_b200.so; raises (never falls back) when the extension is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2110_11226_b200.build` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib
