"""ctypes binding of the C-ABI engine (`include/autoplan_b200.h`).

The engine has no CPU fallback: importing this module succeeds on a CPU-only
machine (so the package and its host logic can be used and tested), but any
compute call raises `EngineUnavailable` unless the in-tree
`libautoplan_b200.so` is built and a CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

# AP_LIB_PATH: developer override to A/B an alternative build of the same engine
LIB_PATH = Path(os.environ.get("AP_LIB_PATH") or Path(__file__).resolve().parent / "libautoplan_b200.so")

AP_OK = 0
AP_ERR_INVALID = -1
AP_ERR_CUDA = -2
AP_ERR_UNSUPPORTED = -3
AP_ERR_INFEASIBLE = -4

OUTCOME_COMPLETE = 0
OUTCOME_INCOMPLETE = 1
OUTCOME_CONFLICT = 2


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library missing or no GPU)."""


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class GraphDesc(ctypes.Structure):
    _fields_ = [
        ("num_instructions", ctypes.c_int32),
        ("opcode", ctypes.c_void_p),
        ("rank", ctypes.c_void_p),
        ("dims_offset", ctypes.c_void_p),
        ("dims", ctypes.c_void_p),
        ("operand_offset", ctypes.c_void_p),
        ("operands", ctypes.c_void_p),
        ("gte_element", ctypes.c_void_p),
    ]


class GraphInfo(ctypes.Structure):
    _fields_ = [
        ("num_slots", ctypes.c_int64),
        ("num_classes", ctypes.c_int32),
        ("num_links", ctypes.c_int32),
        ("num_implications", ctypes.c_int64),
        ("num_forced", ctypes.c_int32),
    ]


class Topology(ctypes.Structure):
    _fields_ = [
        ("num_servers", ctypes.c_int32),
        ("gpus_per_server", ctypes.c_int32),
        ("intra_bw", ctypes.c_double),
        ("inter_bw", ctypes.c_double),
    ]

    @classmethod
    def of(cls, topo) -> "Topology":
        return cls(int(topo.num_servers), int(topo.gpus_per_server), float(topo.intra_bw), float(topo.inter_bw))


class PipeDesc(ctypes.Structure):
    _fields_ = [
        ("num_forward", ctypes.c_int32),
        ("cost_ms", ctypes.c_void_p),
        ("out_bytes", ctypes.c_void_p),
        ("last_use", ctypes.c_void_p),
        ("num_vars", ctypes.c_int32),
        ("var_anchor", ctypes.c_void_p),
        ("var_bytes", ctypes.c_void_p),
    ]


# every symbol the header declares: name -> (restype, argtypes)
_VP = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_F64 = ctypes.c_double
_F32 = ctypes.c_float
_U64 = ctypes.c_uint64
_TOPO = ctypes.POINTER(Topology)


class ParityLoopDesc(ctypes.Structure):
    """ap_parity_loop (include/autoplan_b200.h): the device search loop's buffers."""

    _fields_ = [
        ("ctl", ctypes.c_void_p), ("dctl", ctypes.c_void_p), ("rng", ctypes.c_void_p),
        ("n", ctypes.c_int32), ("ld", ctypes.c_int32), ("num_actions", ctypes.c_int32),
        ("seeds", ctypes.c_void_p), ("seeds_try", ctypes.c_void_p), ("decided", ctypes.c_void_p),
        ("status", ctypes.c_void_p), ("outcome", ctypes.c_void_p), ("order", ctypes.c_void_p),
        ("t_seeds", ctypes.c_void_p), ("t_decided", ctypes.c_void_p), ("state", ctypes.c_void_p),
        ("r_states", ctypes.c_void_p), ("r_next", ctypes.c_void_p), ("r_ld", ctypes.c_int64), ("cap", ctypes.c_int64),
        ("r_actions", ctypes.c_void_p), ("r_rewards", ctypes.c_void_p), ("r_done", ctypes.c_void_p),
        ("r_mask", ctypes.c_void_p), ("r_prio", ctypes.c_void_p),
        ("eps_start", ctypes.c_double), ("eps_final", ctypes.c_double), ("eps_decay", ctypes.c_int64),
        ("best_row", ctypes.c_void_p), ("log_action", ctypes.c_void_p), ("log_reward", ctypes.c_void_p),
        ("log_pos", ctypes.c_void_p), ("log_decided", ctypes.c_void_p), ("ep_conflict", ctypes.c_void_p),
        ("ep_len", ctypes.c_void_p), ("ep_return", ctypes.c_void_p), ("loss_log", ctypes.c_void_p),
        ("loss_cap", ctypes.c_int64),
        ("learn_gate", ctypes.c_int64), ("r_scaled", ctypes.c_void_p), ("pstat", ctypes.c_void_p),
        ("per_alpha", ctypes.c_double),
        ("early_sample", ctypes.c_int64),
    ]


_PL = ctypes.POINTER(ParityLoopDesc)


class FusedLearnDesc(ctypes.Structure):
    """ap_fused_learn (include/autoplan_b200.h): one fused DQN learn step."""

    _fields_ = [
        ("L", ctypes.c_int32), ("dims", ctypes.c_int32 * 6), ("w_off", ctypes.c_int64 * 5),
        ("b_off", ctypes.c_int64 * 5), ("batch", ctypes.c_int32), ("params", ctypes.c_void_p),
        ("target", ctypes.c_void_p), ("r_states", ctypes.c_void_p), ("r_next", ctypes.c_void_p),
        ("r_ld", ctypes.c_int64), ("r_actions", ctypes.c_void_p), ("r_rewards", ctypes.c_void_p),
        ("r_done", ctypes.c_void_p), ("r_mask", ctypes.c_void_p), ("r_prio", ctypes.c_void_p),
        ("idx", ctypes.c_void_p), ("weights", ctypes.c_void_p), ("gamma", ctypes.c_float),
        ("huber_delta", ctypes.c_float), ("grad", ctypes.c_void_p), ("m", ctypes.c_void_p), ("v", ctypes.c_void_p),
        ("nparams", ctypes.c_int64), ("lr", ctypes.c_float), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
        ("eps", ctypes.c_float), ("correct1", ctypes.c_float), ("correct2", ctypes.c_float),
        ("ctab", ctypes.c_void_p), ("ctl", ctypes.c_void_p), ("t_offset", ctypes.c_int64),
        ("wt", ctypes.c_void_p * 5), ("wt_ld", ctypes.c_int64 * 5), ("td", ctypes.c_void_p),
        ("loss", ctypes.c_void_p), ("workspace", ctypes.c_void_p), ("barrier", ctypes.c_void_p),
        ("trace", ctypes.c_void_p),
        ("gate", ctypes.c_int64),
        ("tail_ctl", ctypes.c_void_p), ("loss_log", ctypes.c_void_p), ("loss_cap", ctypes.c_int64),
        ("sync_every", ctypes.c_int32), ("sync_n", ctypes.c_int32), ("sync_src", ctypes.c_void_p * 6),
        ("sync_dst", ctypes.c_void_p * 6), ("sync_count", ctypes.c_int64 * 6),
        ("r_scaled", ctypes.c_void_p), ("pstat", ctypes.c_void_p), ("per_alpha", ctypes.c_double),
        ("lazy_wt0", ctypes.c_int32), ("rng_from", ctypes.c_void_p), ("rng_to", ctypes.c_void_p),
    ]
PL = {"STEP": 0, "SLOT": 1, "SIZE": 2, "TRAIN": 3, "EPISODES": 4, "BUDGET": 5, "MAX_STEPS": 6, "POS": 7,
      "EP_STEPS": 8, "BEST_PART": 9, "BEST_EP": 10, "SYNC": 11, "T_POS": 12, "EP_BASE": 13, "TRAIN0": 14,
      "LOSS_BAD": 15, "TAB_BASE": 16, "ACTIVE": 17, "GEN": 18, "ACK": 19, "FAULT": 20, "WORDS": 32}
SIGNATURES: dict[str, tuple] = {
    "ap_graph_create": (ctypes.c_int, [ctypes.POINTER(GraphDesc), ctypes.POINTER(_VP)]),
    "ap_graph_destroy": (ctypes.c_int, [_VP]),
    "ap_graph_get_info": (ctypes.c_int, [_VP, ctypes.POINTER(GraphInfo)]),
    "ap_graph_export": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "ap_decision_create": (ctypes.c_int, [_VP, _VP, _VP, _I32, ctypes.POINTER(_VP)]),
    "ap_decision_destroy": (ctypes.c_int, [_VP]),
    "ap_propagate_batch": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _VP, _VP]),
    "ap_propagate_batch_packed": (ctypes.c_int, [_VP, _VP, _VP, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _VP, _VP]),
    "ap_parity_act": (ctypes.c_int, [_PL, _VP, _VP, _VP]),
    "ap_parity_post": (ctypes.c_int, [_PL, _VP, _VP]),
    "ap_parity_act_fused": (ctypes.c_int, [_PL, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_parity_sample": (ctypes.c_int, [_PL, _I32, _F64, _F64, _VP, _VP, _VP, _VP, _VP, _I32, _VP]),
    "ap_parity_learn_tail": (ctypes.c_int, [_PL, _VP, _I32, _VP]),
    "ap_per_scaled": (ctypes.c_int, [_VP, _I64, _F64, _VP, _VP, _VP]),
    "ap_parity_target_sync": (ctypes.c_int, [_VP, _I32, _VP, _VP, _VP, _VP]),
    "ap_dqn_adam_tab": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _F32, _F32, _F32, _F32, _VP, _VP, _I64, _VP]),
    "ap_loop_graph_create": (ctypes.c_int, [_VP, _VP, _VP, _I64, ctypes.POINTER(_VP)]),
    "ap_loop_graph_launch": (ctypes.c_int, [_VP, _VP]),
    "ap_loop_graph_destroy": (ctypes.c_int, [_VP]),
    "ap_pcg64_host_draws": (ctypes.c_int, [_VP, _VP, _I32, _VP]),
    "ap_mlp_fused_workspace": (ctypes.c_int64, [_I32, _VP, _I32, _I32]),
    "ap_dqn_learn_fused": (ctypes.c_int, [ctypes.POINTER(FusedLearnDesc), _VP]),
    "ap_mlp_forward_fused": (ctypes.c_int, [_I32, _VP, _VP, _VP, _VP, _VP, _I64, _I32, _VP, _VP, _VP, _VP]),
    "ap_generate_envs": (ctypes.c_int, [_I32, _VP, _I64, _I32, _I32, _VP, _VP]),
    "ap_np_samples_host": (ctypes.c_int, [_VP, _I32, _I64, _I64, _F64, _VP]),
    "ap_generate_envs_host": (ctypes.c_int, [_I32, _VP, _I64, _I32, _I32, _VP]),
    "ap_propagate_trace": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_pipe_create": (ctypes.c_int, [ctypes.POINTER(PipeDesc), ctypes.POINTER(_VP)]),
    "ap_pipe_destroy": (ctypes.c_int, [_VP]),
    "ap_pipe_candidates": (ctypes.c_int, [_VP, _TOPO, _I32, _I32, _VP, _VP]),
    "ap_pipe_metrics": (ctypes.c_int, [_VP, _VP, _I64, _I32, _F64, _VP, _VP, _VP, _VP, _VP]),
    "ap_pipe_metrics_bound": (ctypes.c_int, [_VP, _VP, _I32, _VP, _I64, _I32, _F64, _VP, _VP, _VP, _VP, _VP]),
    "ap_pipe_length": (ctypes.c_int, [_TOPO, _I32, _I32, _I64, _VP, _VP, _VP, _VP, _I32, _F64, _F64, _I32, _VP, _VP,
                                      _VP]),
    "ap_pipe_train_state": (ctypes.c_int, [_VP, _TOPO, _VP, _I32, _VP, _I32, _VP, _I64, _F64, _VP, _VP]),
    "ap_pipe_train_table": (ctypes.c_int, [_VP, _VP, _I32, _VP]),
    "ap_generate_uniform_envs": (ctypes.c_int, [_VP, _I64, _I32, _I32, _VP, _VP]),
    "ap_pipe_train_state_ex": (ctypes.c_int, [_VP, _TOPO, _VP, _I32, _VP, _I32, _VP, _I64, _F64, _VP, _VP, _I64, _VP, _I64,
                                              _VP]),
    "ap_infer_length": (ctypes.c_int, [_VP, _I32, _TOPO, _I32, _I32, _VP, _VP, _I64, _VP, _VP]),
    "ap_infer_search": (ctypes.c_int, [_VP, _I32, _TOPO, _I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_gemm_tf32": (ctypes.c_int, [_VP, _I64, _I32, _VP, _I64, _I32, _VP, _I64, _I32, _I32, _I32, _VP, _I32, _I32,
                                    _VP]),
    "ap_dqn_dueling": (ctypes.c_int, [_VP, _I64, _VP, _I64, _I32, _I32, _VP]),
    "ap_dqn_act": (ctypes.c_int, [_VP, _I64, _VP, _I64, _I32, _I32, ctypes.c_float, ctypes.c_uint64, _VP, _VP]),
    "ap_dqn_td": (ctypes.c_int, [_VP, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _I64, _VP, _I32, _I32, ctypes.c_float,
                                 ctypes.c_float, _VP, _I64, _VP, _VP, _VP]),
    "ap_dqn_td_ring": (ctypes.c_int, [_VP, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _I64, _VP, _I32, _I32, _F32, _F32,
                                      _VP, _I64, _VP, _I64, _VP, _VP, _VP]),
    "ap_dqn_head_forward": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I32, _I32, _I32, _VP, _I64, _VP]),
    "ap_dqn_relu_backward_t": (ctypes.c_int, [_VP, _I64, _VP, _I64, _I32, _I32, _VP, _I64, _VP]),
    "ap_transpose_batch": (ctypes.c_int, [_I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_dqn_relu_backward": (ctypes.c_int, [_VP, _VP, _I64, _VP]),
    "ap_dqn_colsum": (ctypes.c_int, [_VP, _I64, _I32, _I32, _VP, _VP]),
    "ap_probe_fp64_add": (ctypes.c_int, [_I32, _I64, _VP, _VP]),
    "ap_dqn_head_backward_dueling": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _VP, _VP, _I64, _VP,
                                                     _I64, _VP]),
    "ap_dqn_head_backward": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _VP, _I64, _VP, _I64,
                                            _VP]),
    "ap_dqn_adam": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                   ctypes.c_float, ctypes.c_float, ctypes.c_float, _VP]),
    "ap_per_sample": (ctypes.c_int, [_VP, _I32, _F64, _F64, _VP, _I32, _VP, _VP, _VP, _VP]),
    "ap_per_update": (ctypes.c_int, [_VP, _VP, _VP, _I32, _VP]),
    "ap_gather_rows_pair": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I64, _VP, _I64, _VP, _I32, _I32, _VP]),
    "ap_gather_rows": (ctypes.c_int, [_VP, _I64, _VP, _I32, _I32, _VP, _I64, _VP]),
    "ap_vec_apply": (ctypes.c_int, [_VP, _I64, _VP, _VP, _I32, _VP]),
    "ap_pack_slots2": (ctypes.c_int, [_VP, _I64, _I64, _I64, _VP, _I64, _VP]),
    "ap_vec_post": (ctypes.c_int, [_I32, _I32, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I64, _VP, _VP, _VP, _VP,
                                   _I32, _VP, _VP, _VP, _VP, _VP]),
    "ap_vec_track_best": (ctypes.c_int, [_I32, _I32, _I64, _VP, _VP, _VP, _VP, _VP, _I64, _VP, _I32, _I32, _VP, _VP,
                                         _VP, _VP, _VP]),
    "ap_dqn_act_ctl": (ctypes.c_int, [_VP, _I64, _VP, _I64, _I32, _I32, _F32, _F32, _I64, _VP, _VP, _VP]),
    "ap_dp_allreduce_adam": (ctypes.c_int, [_I32, _I32, _VP, _VP, _VP, _I64, _VP, _VP, _VP, _F32, _F32, _F32, _F32,
                                            _VP, _VP, _VP]),
    "ap_dqn_adam_ctl_t": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _F32, _F32, _F32, _F32, _VP, _I32, _VP, _VP, _VP,
                                         _VP, _VP, _VP]),
    "ap_gemm_tf32_adam": (ctypes.c_int, [_VP, _I64, _VP, _I64, _VP, _I64, _I32, _I32, _I32, _VP, _VP, _VP, _VP, _I32,
                                         _F32, _F32, _F32, _F32, _VP, _I64, _I32, _VP]),
    "ap_dqn_adam_ctl_t_adv": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _F32, _F32, _F32, _F32, _VP, _I32, _VP, _VP,
                                             _VP, _VP, _VP, _I32, _VP]),
    "ap_per_update_scaled_ctl": (ctypes.c_int, [_VP, _VP, _VP, _I32, _F64, _VP, _VP]),
    "ap_dqn_adam_ctl": (ctypes.c_int, [_VP, _VP, _VP, _VP, _I64, _F32, _F32, _F32, _F32, _VP, _VP]),
    "ap_per_push_ctl": (ctypes.c_int, [_I32, _I32, _I32, _I64, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                       _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_per_sample_ctl": (ctypes.c_int, [_VP, _I64, _F64, _I32, _U64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_vec_pipe_apply": (ctypes.c_int, [_I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_vec_pipe_post": (ctypes.c_int, [_I32, _I32, _I32, _I32, _VP, _VP, _VP, _I32, _VP, _VP, _VP, _VP, _VP, _VP,
                                        _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I32, _I32, _VP]),
    "ap_vec_infer_apply": (ctypes.c_int, [_I32, _I32, _I32, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "ap_vec_infer_post": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                         _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I32, _I32,
                                         _VP]),
    "ap_vec_ctl_advance": (ctypes.c_int, [_VP, _I32, _I64, _I64, _VP]),
    "ap_per_push": (ctypes.c_int, [_I32, _I32, _I32, _I64, _I64, _VP, _VP, _I64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                   _VP, _VP, _VP, _VP, _VP]),
    "ap_per_sample_fast": (ctypes.c_int, [_VP, _I32, _F64, _F64, _VP, _I32, _VP, _VP, _VP, _VP, _VP]),
    "ap_per_update_scaled": (ctypes.c_int, [_VP, _VP, _VP, _I32, _F64, _VP]),
    "ap_last_error": (ctypes.c_char_p, []),
    "ap_version": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None):
    """Load the engine library and bind its C-ABI signatures (no GPU needed).  AP_LIB_PATH
    names another build of the same library (profiling variants)."""
    global _lib
    path = path or os.environ.get("AP_LIB_PATH") or LIB_PATH
    with _lock:
        if _lib is None:
            if not Path(path).exists():
                raise EngineUnavailable(
                    f"{path} is not built; run `python -m paper_2007_04069_b200.build` (nvcc, sm_100a)"
                )
            lib = ctypes.CDLL(str(path))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def require_device():
    """The library plus a CUDA device, or EngineUnavailable."""
    import torch

    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return load_library()


def check(rc: int) -> None:
    if rc != AP_OK:
        msg = _lib.ap_last_error().decode(errors="replace") if _lib is not None else "unknown"
        raise NativeError(rc, msg)


def ptr(a) -> ctypes.c_void_p | None:
    """Raw pointer of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


def stream_handle(stream=None) -> ctypes.c_void_p:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class DeviceGraph:
    """Per-graph engine tables (ap_graph_t).

    The rule compile runs on the host at construction (so `export()` works
    without a GPU); the tables are uploaded to `device_index` on first use.
    """

    def __init__(self, flat, device_index: int | None = None):
        lib = load_library()
        self.flat = flat
        self.device_index = device_index
        self._keep = [
            np.ascontiguousarray(a) if a.size else np.zeros(1, dtype=a.dtype)
            for a in (flat.opcode, flat.rank, flat.dims_offset, flat.dims, flat.operand_offset, flat.operands,
                      flat.gte_element)
        ]
        desc = GraphDesc(flat.num_instructions, *[a.ctypes.data for a in self._keep])
        handle = ctypes.c_void_p()
        check(lib.ap_graph_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        info = GraphInfo()
        check(lib.ap_graph_get_info(handle, ctypes.byref(info)))
        self.num_slots = int(info.num_slots)
        self.num_classes = int(info.num_classes)
        self.num_links = int(info.num_links)
        self.num_implications = int(info.num_implications)
        self.num_forced = int(info.num_forced)
        self._decisions: dict[tuple, DeviceDecision] = {}

    def export(self) -> dict[str, np.ndarray]:
        """Host copies of the compiled tables (tests / tooling)."""
        cls = np.empty(max(self.num_slots, 1), dtype=np.int32)
        forced = np.empty(max(self.num_classes, 1), dtype=np.uint8)
        off = np.empty(self.num_classes + 1, dtype=np.int32)
        tgt = np.empty(max(self.num_implications, 1), dtype=np.int32)
        check(_lib.ap_graph_export(self.handle, ptr(cls), ptr(forced), ptr(off), ptr(tgt)))
        return {
            "class_of_slot": cls[: self.num_slots],
            "class_forced": forced[: self.num_classes],
            "imp_offset": off,
            "imp_target": tgt[: self.num_implications],
        }

    def decision(self, slots: np.ndarray, is_candidate: np.ndarray) -> "DeviceDecision":
        key = (slots.tobytes(), is_candidate.tobytes())
        dec = self._decisions.get(key)
        if dec is None:
            dec = DeviceDecision(self, slots, is_candidate)
            self._decisions[key] = dec
        return dec

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            for d in self.__dict__.get("_decisions", {}).values():
                d.close()
            _lib.ap_graph_destroy(h)
            self.handle = None


class DeviceDecision:
    """A decision set (ap_decision_t): seed / candidate slot positions."""

    def __init__(self, graph: DeviceGraph, slots: np.ndarray, is_candidate: np.ndarray):
        self.graph = graph
        self.slots = np.ascontiguousarray(slots, dtype=np.int64)
        self.is_candidate = np.ascontiguousarray(is_candidate, dtype=np.uint8)
        self.n = int(self.slots.shape[0])
        handle = ctypes.c_void_p()
        check(_lib.ap_decision_create(graph.handle, ptr(self.slots) if self.n else None,
                                      ptr(self.is_candidate) if self.n else None, self.n, ctypes.byref(handle)))
        self.handle = handle

    def close(self):
        if getattr(self, "handle", None) is not None and _lib is not None:
            _lib.ap_decision_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.close()
