"""ctypes binding of include/pvi_b200.h (the C ABI of libpvi_b200.so).

The shared library is built in-tree (paper_2303_10672_b200/lib/) by
`__graft_entry__.build()`.  There is no fallback: if the library cannot be
loaded every entry point raises, so a missing build fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libpvi_b200.so")

_vp = C.c_void_p


class ScenarioAParams(C.Structure):
    _fields_ = [("useful_life", C.c_int), ("lead_time", C.c_int), ("issuing", C.c_int),
                ("max_order", C.c_int), ("max_demand", C.c_int), ("unit_cost", C.c_double),
                ("holding_cost", C.c_double), ("shortage_cost", C.c_double),
                ("wastage_cost", C.c_double), ("demand_mean", C.c_double),
                ("demand_cv", C.c_double), ("discount_factor", C.c_double)]


class ScenarioBParams(C.Structure):
    _fields_ = [("useful_life", C.c_int), ("demand_mean_a", C.c_double),
                ("demand_mean_b", C.c_double), ("max_order_a", C.c_int),
                ("max_order_b", C.c_int), ("unit_cost_a", C.c_double),
                ("unit_cost_b", C.c_double), ("revenue_a", C.c_double),
                ("revenue_b", C.c_double), ("substitution_prob", C.c_double),
                ("discount_factor", C.c_double)]


C_MAX_LIFE = 12


class ScenarioCParams(C.Structure):
    _fields_ = [("useful_life", C.c_int), ("max_order", C.c_int), ("max_demand", C.c_int),
                ("fixed_order_cost", C.c_double), ("holding_cost", C.c_double),
                ("shortage_cost", C.c_double), ("wastage_cost", C.c_double),
                ("discount_factor", C.c_double), ("demand_successes", C.c_double * 7),
                ("demand_means", C.c_double * 7),
                ("life_intercepts", C.c_double * (C_MAX_LIFE - 1)),
                ("life_slopes", C.c_double * (C_MAX_LIFE - 1))]


class ModelInfo(C.Structure):
    _fields_ = [("scenario", C.c_int), ("state_count", C.c_uint64),
                ("action_count", C.c_uint32), ("outcome_count", C.c_uint64),
                ("discount", C.c_double), ("default_convergence_test", C.c_int),
                ("periodicity", C.c_int), ("state_arity", C.c_uint32),
                ("action_arity", C.c_uint32), ("products", C.c_int),
                ("terms_per_sweep", C.c_double), ("max_order_a", C.c_int),
                ("max_order_b", C.c_int), ("factored_fmas", C.c_double),
                ("receipt_exogenous", C.c_int)]


class ViConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("gamma", C.c_double), ("has_gamma", C.c_int),
                ("max_iterations", C.c_uint64), ("fixed_iterations", C.c_uint64),
                ("checkpoint_every", C.c_uint64), ("checkpoint_path", C.c_char_p),
                ("precision", C.c_int), ("convergence_test", C.c_int),
                ("max_states", C.c_uint64), ("device", C.c_int),
                ("algorithm", C.c_int), ("loop", C.c_int), ("l2_persist", C.c_int)]


class ViStats(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("converged", C.c_int),
                ("wall_seconds", C.c_double), ("sweep_seconds", C.c_double),
                ("sweeps", C.c_uint64), ("span_lo", C.c_double), ("span_hi", C.c_double),
                ("terms_per_sweep", C.c_double), ("graph_sweeps", C.c_uint64),
                ("l2_window_bytes", C.c_uint64), ("l2_hit_ratio", C.c_double)]


class RolloutConfigC(C.Structure):
    _fields_ = [("horizon_days", C.c_int), ("warmup_days", C.c_int), ("n_rollouts", C.c_int),
                ("base_seed", C.c_uint64), ("device", C.c_int)]


class RolloutSummaryC(C.Structure):
    _fields_ = [("ret", C.c_double), ("service_pct", C.c_double * 2),
                ("wastage_pct", C.c_double * 2), ("holding_mean", C.c_double * 2)]


class EvaluationC(C.Structure):
    _fields_ = [("ret_mean", C.c_double), ("ret_sd", C.c_double),
                ("service_mean", C.c_double * 2), ("service_sd", C.c_double * 2),
                ("wastage_mean", C.c_double * 2), ("wastage_sd", C.c_double * 2),
                ("holding_mean", C.c_double * 2), ("holding_sd", C.c_double * 2),
                ("products", C.c_int), ("n_rollouts", C.c_int)]


class SimoptConfigC(C.Structure):
    _fields_ = [("sampler", C.c_int), ("population", C.c_int), ("max_generations", C.c_int),
                ("patience", C.c_int), ("crossover_rate", C.c_double),
                ("mutation_rate", C.c_double), ("seed", C.c_uint64),
                ("rollouts_per_candidate", C.c_int), ("horizon_days", C.c_int),
                ("warmup_days", C.c_int), ("base_seed", C.c_uint64), ("device", C.c_int),
                ("score_batch", C.c_void_p), ("score_user", C.c_void_p)]


# int (*)(void* user, const int* candidates, int n, int dimension, double* means, double* sds)
SCORE_BATCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_int, C.c_int,
                             C.POINTER(C.c_double), C.POINTER(C.c_double))


class ScoredCandidateC(C.Structure):
    _fields_ = [("generation", C.c_int), ("values", C.c_int * 14), ("mean", C.c_double),
                ("sd", C.c_double)]


class PolicyC(C.Structure):
    _fields_ = [("kind", C.c_int), ("table", C.POINTER(C.c_uint32)),
                ("params", C.c_int * 14), ("n_params", C.c_int)]


# Every symbol include/pvi_b200.h declares, with its ctypes signature.
_E = [C.c_char_p, C.c_size_t]
SIGNATURES = {
    "pvi_exit_code": (C.c_int, [C.c_int]),
    "pvi_version": (C.c_char_p, []),
    "pvi_device_count": (C.c_int, []),
    "pvi_scenario_a_defaults": (None, [_vp]),
    "pvi_scenario_b_defaults": (None, [_vp]),
    "pvi_scenario_c_defaults": (None, [_vp]),
    "pvi_model_create_a": (C.c_int, [_vp, _vp] + _E),
    "pvi_model_create_b": (C.c_int, [_vp, _vp] + _E),
    "pvi_model_create_c": (C.c_int, [_vp, _vp] + _E),
    "pvi_model_create_tabular": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double,
                                           _vp, _vp, _vp, _vp, _vp] + _E),
    "pvi_model_create_preset": (C.c_int, [C.c_char_p, _vp, _vp, _vp] + _E),
    "pvi_model_destroy": (None, [_vp]),
    "pvi_model_get_info": (C.c_int, [_vp, _vp]),
    "pvi_model_fingerprint_material": (C.c_int, [_vp, C.c_char_p, C.c_size_t]),
    "pvi_model_fingerprint": (C.c_int, [_vp, _vp]),
    "pvi_model_table": (C.c_int, [_vp, C.c_char_p, _vp, _vp]),
    "pvi_model_decode": (C.c_int, [_vp, C.c_uint64, _vp]),
    "pvi_model_encode": (C.c_int, [_vp, _vp, _vp] + _E),
    "pvi_model_transition": (C.c_int, [_vp, C.c_uint64, C.c_uint32, C.c_uint64, _vp, _vp] + _E),
    "pvi_model_outcome_probability": (C.c_int, [_vp, C.c_uint64, C.c_uint32, C.c_uint64, _vp]),
    "pvi_model_initial_values": (C.c_int, [_vp, _vp] + _E),
    "pvi_vi_config_defaults": (None, [_vp]),
    "pvi_model_set_algorithm": (C.c_int, [_vp, C.c_int]),
    "pvi_vi_solve": (C.c_int, [_vp, _vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp, _vp] + _E),
    "pvi_vi_backup": (C.c_int, [_vp, C.c_int, C.c_double, _vp, C.c_uint64, C.c_uint64, _vp,
                                _vp] + _E),
    "pvi_q_rows": (C.c_int, [_vp, C.c_int, C.c_double, _vp, C.c_uint64, C.c_uint64, _vp] + _E),
    "pvi_check_convergence": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_int, C.c_double,
                                        C.c_double, C.c_uint64, _vp] + _E),
    "pvi_vi_sweep_device": (C.c_int, [_vp, C.c_int, C.c_double, _vp, _vp, _vp, C.c_uint64,
                                      C.c_uint64, C.c_int, _vp, C.c_int, C.c_int, _vp,
                                      _vp] + _E),
    "pvi_partition": (C.c_int, [_vp, C.c_int, _vp]),
    "pvi_sweep_read_runs": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)]),
    "pvi_vi_sweep_device_peers": (C.c_int, [_vp, C.c_int, C.c_double, _vp, _vp, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp, _vp, _vp, C.c_char_p, C.c_size_t]),
    "pvi_unit_count": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "pvi_unit_partition": (C.c_int, [_vp, C.c_int, _vp]),
    "pvi_unit_runs": (C.c_int, [_vp, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_size_t)]),
    "pvi_vi_sweep_device_units": (C.c_int, [_vp, C.c_int, C.c_double, _vp, _vp, _vp, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _vp, _vp, C.c_int, _vp, _vp, _vp, C.c_char_p, C.c_size_t]),
    "pvi_device_alloc": (C.c_int, [C.c_uint64, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "pvi_device_free": (C.c_int, [_vp]),
    "pvi_ipc_get_handle": (C.c_int, [_vp, _vp, C.c_char_p, C.c_size_t]),
    "pvi_ipc_open": (C.c_int, [_vp, C.POINTER(C.c_void_p), C.c_char_p, C.c_size_t]),
    "pvi_ipc_close": (C.c_int, [_vp]),
    "pvi_policy_csv_format": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    "pvi_policy_csv_parse": (C.c_int, [_vp, _vp, C.c_uint64, _vp, C.c_char_p, C.c_size_t]),
    "pvi_rollout_config_defaults": (None, [_vp]),
    "pvi_sim_evaluate": (C.c_int, [_vp, _vp, C.c_uint32, _vp, _vp, _vp] + _E),
    "pvi_sim_reduce": (C.c_int, [_vp, C.c_uint32, C.c_int, C.c_int, _vp] + _E),
    "pvi_philox_block": (C.c_int, [_vp, _vp, _vp]),
    "pvi_rollout_draws": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, _vp]),
    "pvi_checkpoint_save": (C.c_int, [C.c_char_p, _vp, C.c_uint64, C.c_uint64, _vp] + _E),
    "pvi_checkpoint_load": (C.c_int, [C.c_char_p, _vp, _vp, C.c_uint64, _vp, _vp, _vp] + _E),
    "pvi_sha256": (C.c_int, [_vp, C.c_size_t, _vp]),
    "pvi_simopt_config_defaults": (None, [_vp]),
    "pvi_simopt": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp] + _E),
    "pvi_profile_enable": (C.c_int, [C.c_int]),
    "pvi_profile_sim_read": (C.c_int, [_vp, _vp, _vp]),
    "pvi_profile_read": (C.c_int, [_vp, _vp, _vp]),
}

_lib = None


def load():
    """Load libpvi_b200.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(pvi_b200 has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
