"""ctypes binding of include/morphling.h (argument marshalling only).

Every function here has the same name and argument order as its C counterpart; device
pointers are passed as integers (e.g. `tensor.data_ptr()`), streams as integers
(`torch.cuda.current_stream().cuda_stream`).  A non-zero status raises MorphlingError
carrying the C-ABI code and `mph_last_error()`.  There is no Python fallback: if the
shared library is missing, importing this module fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmorphling.so")

STATUS = {0: "MPH_OK", -1: "MPH_EINVAL", -2: "MPH_ERANGE", -3: "MPH_EDEGENERATE", -4: "MPH_ESTATE",
          -5: "MPH_ENOMEM", -6: "MPH_ECUDA", -7: "MPH_ENCCL", -8: "MPH_EDIVERGED", -9: "MPH_ENOTSUP",
          -10: "MPH_ETIMEOUT"}

EPI_BIAS, EPI_RELU, EPI_ROWSCALE, EPI_MASK, EPI_DROPOUT, EPI_COLSUM, EPI_TF32 = 1, 2, 4, 8, 16, 32, 64
EPI_BF16, EPI_MASK_BF16, EPI_SIGNBITS, EPI_MASK_BITS = 128, 256, 1024, 2048
AGG = {"gcn": 0, "sum": 1, "mean": 2, "max": 3}            # MPH_AGG_*
TAU_PAPER_BP, TAU_B200_BP = 8000, 9500                     # MPH_TAU_PAPER_BP, MPH_TAU_B200_BP
OPT = {"adam": 0, "sgd": 1, "adamw": 2}                    # MPH_OPT_*


class MorphlingError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        super().__init__(f"{fn}: {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class Epilogue(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("row_scale", C.c_void_p), ("bias", C.c_void_p), ("mask_src", C.c_void_p),
                ("ld_mask", C.c_int32), ("mask_scale", C.c_float), ("colsum_out", C.c_void_p),
                ("dropout_p", C.c_float), ("dropout_seed", C.c_uint64), ("dropout_layer", C.c_int32),
                ("dropout_epoch", C.c_int32), ("row0", C.c_int64), ("dropout_epoch_d", C.c_void_p),
                ("bits_out", C.c_void_p), ("ld_bits", C.c_int32)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float)]


class OptimCfg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("weight_decay", C.c_float), ("momentum", C.c_float)]


class GcnDesc(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("dims_h", C.POINTER(C.c_int32)), ("dropout_p", C.c_float),
                ("dropout_seed", C.c_uint64), ("order_policy", C.c_int32), ("aggregator", C.c_int32),
                ("comm_mode", C.c_int32), ("precision", C.c_int32)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      f"(or `python paper_2512_01678_b200/build.py`)")
_lib = C.CDLL(LIB_PATH)

P = C.c_void_p
i32, i64, u64, f32, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_size_t
PP = C.POINTER(C.c_void_p)

# name -> argtypes (all return int status except mph_version / mph_last_error)
_SIGS = {
    "mph_launch_count": [C.POINTER(i64)],
    "mph_device_check": [C.POINTER(i32)],
    "mph_graph_build": [P, P, i64, i32, P, PP],
    "mph_graph_info": [P, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64), C.POINTER(i32)],
    "mph_graph_csr": [P, PP, PP, PP, PP],
    "mph_graph_destroy": [P],
    "mph_features_create": [P, i32, i32, i32, i32, i32, P, PP],
    "mph_features_create_csr": [P, P, P, i32, i32, i32, i32, P, PP],
    "mph_features_info": [P, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32)],
    "mph_features_count": [P, i32, i32, i32, P, C.POINTER(i64)],
    "mph_features_decide": [i64, i64, i64, i32, C.POINTER(i32)],
    "mph_features_csr": [P, PP, PP, PP],
    "mph_features_csc": [P, PP, PP, PP],
    "mph_features_dense": [P, PP, C.POINTER(i32)],
    "mph_features_destroy": [P],
    "mph_spmm": [P, P, i32, i32, P, i32, C.POINTER(Epilogue), P],
    "mph_spmm_signbits_ok": [P, i32, C.POINTER(i32)],
    "mph_spmm_part": [P, i32, P, i32, i32, P, i32, C.POINTER(Epilogue), P],
    "mph_graph_agg_scales": [P, i32, i32, PP, PP],
    "mph_aggregate": [P, i32, i32, P, i32, i32, P, i32, C.POINTER(Epilogue), P],
    "mph_aggregate_max": [P, P, i32, i32, P, i32, P, i32, C.POINTER(Epilogue), P],
    "mph_aggregate_max_backward": [P, P, i32, i32, P, i32, P, i32, C.POINTER(Epilogue), P],
    "mph_gemm_nt": [i32, i32, i32, P, i32, P, i32, P, i32, C.POINTER(Epilogue), P],
    "mph_gemm_tn_workspace": [i32, i32, i32, C.POINTER(sz)],
    "mph_gemm_tn": [i32, i32, i32, P, i32, P, i32, P, i32, P, sz, P],
    "mph_reduce_rows": [P, i32, i32, i32, P, i32, P],
    "mph_sparse_xw": [P, P, i32, i32, P, P, i32, P],
    "mph_sparse_xtg": [P, P, i32, i32, P, i32, P],
    "mph_softmax_ce_workspace": [i32, i32, C.POINTER(sz)],
    "mph_softmax_ce": [P, i32, i32, i32, P, P, i64, P, P, i32, P, P, P, sz, P],
    "mph_adam": [P, P, P, P, i64, C.POINTER(AdamCfg), i32, P],
    "mph_optim_step": [P, P, P, P, i64, C.POINTER(OptimCfg), i32, P],
    "mph_xavier_fill": [P, i32, i32, i32, u64, i32, P],
    "mph_partition_1d": [P, i32, i32, P],
    "mph_partition_greedy": [P, i32, i32, P, P],
    "mph_partition_components": [P, P, i32, i32, P, C.POINTER(i32)],
    "mph_partition_hierarchical": [P, P, i32, i32, P, C.POINTER(i32)],
    "mph_relabel": [P, i32, i32, P, P],
    "mph_partition_stats": [P, P, i32, P, i32, P],
    "mph_plan_create": [P, P, i32, P, i32, i32, PP],
    "mph_plan_info": [P, C.POINTER(i32), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)],
    "mph_plan_arrays": [P, PP, PP, PP, PP, PP, PP, PP, PP, PP],
    "mph_plan_destroy": [P],
    "mph_graph_from_plan": [P, P, PP],
    "mph_comm_unique_id": [P],
    "mph_comm_create": [P, i32, i32, PP],
    "mph_comm_info": [P, C.POINTER(i32), C.POINTER(i32)],
    "mph_comm_destroy": [P],
    "mph_halo_exchange": [P, P, P, i32, i32, P],
    "mph_allreduce_sum": [P, P, i64, i32, P],
    "mph_gcn_create": [P, P, C.POINTER(GcnDesc), P, P, PP],
    "mph_gcn_param_layout": [P, C.POINTER(i64), P, P],
    "mph_gcn_buffers": [P, PP, PP, PP, PP],
    "mph_gcn_init_xavier": [P, u64, P],
    "mph_gcn_params_updated": [P, P],
    "mph_gcn_upload_features": [P, P, i32, P],
    "mph_gcn_upload_features_async": [P, P, i32, P, P],
    "mph_gcn_set_labels": [P, P, P, i64],
    "mph_profile_enable": [i32],
    "mph_probe_gather": [P, i64, i32, P, i64, P, P],
    "mph_probe_l2_stream": [P, i64, i32, P, P],
    "mph_profile_read": [i32, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "mph_gcn_forward": [P, i32, P],
    "mph_gcn_loss": [P, P, P],
    "mph_gcn_backward": [P, P],
    "mph_gcn_adam": [P, C.POINTER(AdamCfg), i32, P],
    "mph_gcn_train_epoch": [P, i32, C.POINTER(AdamCfg), P, P],
    "mph_gcn_graph_capture": [P, C.POINTER(AdamCfg), i32, P],
    "mph_gcn_optim_step": [P, C.POINTER(OptimCfg), i32, P],
    "mph_gcn_train_epoch_opt": [P, i32, C.POINTER(OptimCfg), P, P],
    "mph_gcn_graph_capture_opt": [P, C.POINTER(OptimCfg), i32, P],
    "mph_gcn_graph_replay": [P, P],
    "mph_gcn_graph_state": [P, PP, PP],
    "mph_gcn_tensor": [P, i32, i32, PP, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)],
    "mph_gcn_info": [P, P, C.POINTER(i32)],
    "mph_set_allocator": [P, P, P],
    "mph_graph_localize": [P, P, i32, i32, P, PP],
    "mph_halo_plan": [P, i32, PP, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)],
    "mph_gemm": [i32, i32, i32, P, i32, i32, P, i32, i32, P, i32, i32, C.c_uint32, P],
    "mph_gcn_workspace_size": [P, C.POINTER(sz)],
    "mph_gcn_bind": [P, P, P, P, P, P, sz],
    "mph_adam_step": [P, C.POINTER(AdamCfg), i32, P],
    "mph_gcn_p2p_export": [P, P],
    "mph_gcn_p2p_open": [P, P, i32, P],
    "mph_gcn_p2p_status": [P, C.POINTER(i32), C.POINTER(i64), P],
    "mph_gcn_destroy": [P],
}

COMM = {"nccl": 0, "p2p": 1}
PREC = {"tf32": 0, "bf16": 1}
P2P_BLOB_BYTES = 512

EXPORTED = ["mph_version", "mph_last_error"] + list(_SIGS)

_lib.mph_version.restype = C.c_int
_lib.mph_version.argtypes = []
_lib.mph_last_error.restype = C.c_char_p
_lib.mph_last_error.argtypes = []


def _wrap(name, argtypes):
    f = getattr(_lib, name)
    f.argtypes = argtypes
    f.restype = C.c_int

    def call(*args):
        rc = f(*args)
        if rc != 0:
            raise MorphlingError(rc, name, _lib.mph_last_error().decode(errors="replace"))
        return rc

    call.__name__ = name
    call.__doc__ = f"{name}{tuple(a.__name__ if hasattr(a, '__name__') else str(a) for a in argtypes)} -> status"
    return call


for _n, _a in _SIGS.items():
    globals()[_n] = _wrap(_n, _a)


def mph_version() -> int:
    return _lib.mph_version()


def mph_last_error() -> str:
    return _lib.mph_last_error().decode(errors="replace")


def launch_count() -> int:
    c = i64(0)
    mph_launch_count(C.byref(c))  # noqa: F821
    return c.value


def raw():
    """The underlying ctypes.CDLL (for symbol inspection)."""
    return _lib
