"""ctypes loader for lib/libdsx.so (the dsx C-ABI, include/dsx.h).

Fails loudly when the native library is missing: there is no Python or CPU
fallback for anything the C-ABI does.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PKG_DIR, "lib")
DSX_PATH = os.path.join(LIB_DIR, "libdsx.so")
DREAMSCHED_PATH = os.path.join(LIB_DIR, "libdreamsched.so")

DSX_OK, DSX_ERR_ARGUMENT, DSX_ERR_STATE, DSX_ERR_CUDA, DSX_ERR_NCCL = range(5)
DSX_F64, DSX_F32, DSX_BF16 = 0, 1, 2
DSX_OPT_SGD, DSX_OPT_MOMENTUM, DSX_OPT_ADAM = 0, 1, 2
DSX_EPI_F32, DSX_EPI_BIAS_ACT, DSX_EPI_DRELU, DSX_EPI_ADD, DSX_EPI_BIAS_ADD_ACT, DSX_EPI_ADD_DRELU = 0, 1, 2, 3, 4, 5
DSX_SYNC_PAIRWISE, DSX_SYNC_NCCL_AVG = 0, 1


class DsxError(RuntimeError):
    def __init__(self, status: int, where: str, message: str):
        super().__init__(f"{where}: [{status}] {message}")
        self.status = status


class LabDescC(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("dtype", C.c_int),
        ("workers_total", C.c_int),
        ("worker_begin", C.c_int),
        ("workers_local", C.c_int),
        ("dim", C.c_uint64),
        ("layers", C.c_int),
        ("block_sizes", C.POINTER(C.c_uint64)),
        ("curvature", C.POINTER(C.c_double)),
        ("optimum", C.POINTER(C.c_double)),
        ("noise_sigma", C.c_double),
    ]


class GemmDescC(C.Structure):
    _fields_ = [
        ("dtype", C.c_int), ("M", C.c_int), ("N", C.c_int), ("K", C.c_int), ("batch", C.c_int),
        ("a_mn", C.c_int), ("b_mn", C.c_int),
        ("A", C.c_void_p), ("lda", C.c_longlong), ("strideA", C.c_longlong),
        ("B", C.c_void_p), ("ldb", C.c_longlong), ("strideB", C.c_longlong),
        ("C", C.c_void_p), ("ldc", C.c_longlong), ("strideC", C.c_longlong),
        ("out_dtype", C.c_int), ("epi", C.c_int), ("relu", C.c_int), ("accumulate", C.c_int),
        ("bias", C.c_void_p), ("strideBias", C.c_longlong),
        ("mask", C.c_void_p), ("ldmask", C.c_longlong), ("strideMask", C.c_longlong),
        ("bn", C.c_int), ("stream", C.c_void_p), ("ksplit", C.c_int), ("strideSplit", C.c_longlong),
        ("conv", C.c_int), ("conv_h", C.c_int), ("conv_w", C.c_int), ("conv_images", C.c_int),
        ("conv_cin", C.c_int), ("conv_cout", C.c_int), ("conv_stride", C.c_int), ("conv_k", C.c_int),
        ("mask2", C.c_void_p), ("ldmask2", C.c_longlong), ("strideMask2", C.c_longlong),
    ]


class MlpDescC(C.Structure):
    _fields_ = [
        ("device", C.c_int), ("dtype", C.c_int), ("workers_total", C.c_int), ("worker_begin", C.c_int),
        ("workers_local", C.c_int), ("layers", C.c_int), ("widths", C.POINTER(C.c_int)),
        ("batch", C.c_int), ("optimizer", C.c_int), ("momentum", C.c_double), ("beta1", C.c_double),
        ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
    ]


class CnnDescC(C.Structure):
    _fields_ = [
        ("device", C.c_int), ("dtype", C.c_int), ("workers_total", C.c_int), ("worker_begin", C.c_int),
        ("workers_local", C.c_int), ("width", C.c_int), ("image", C.c_int), ("in_channels", C.c_int),
        ("classes", C.c_int), ("batch", C.c_int), ("optimizer", C.c_int), ("momentum", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
    ]


_dsx = None

_SIGS = {
    "dsx_last_error": ([], C.c_char_p),
    "dsx_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "dsx_warmup": ([], C.c_int),
    "dsx_lab_create": ([C.POINTER(LabDescC), C.POINTER(C.c_void_p)], C.c_int),
    "dsx_lab_destroy": ([C.c_void_p], C.c_int),
    "dsx_lab_set_params": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_lab_get_params": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_lab_fill_params": ([C.c_void_p, C.c_double], C.c_int),
    "dsx_lab_set_all_params": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_get_all_params": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_set_state": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_get_state": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_step_host": ([C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_host_alloc": ([C.c_size_t, C.POINTER(C.c_void_p)], C.c_int),
    "dsx_host_free": ([C.c_void_p], C.c_int),
    "dsx_lab_engine_time": ([C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_int)], C.c_int),
    "dsx_lab_set_rng": ([C.c_void_p, C.c_int, C.c_void_p, C.c_uint64], C.c_int),
    "dsx_lab_get_rng": ([C.c_void_p, C.c_int, C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "dsx_lab_seed_rng": ([C.c_void_p, C.c_uint64], C.c_int),
    "dsx_lab_step": ([C.c_void_p, C.c_double, C.c_void_p], C.c_int),
    "dsx_lab_step_with_noise": ([C.c_void_p, C.c_double, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_last_max_grad_norm_sq": ([C.c_void_p, C.POINTER(C.c_double)], C.c_int),
    "dsx_lab_sync": ([C.c_void_p], C.c_int),
    "dsx_lab_gradient": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_lab_mean_accumulate": ([C.c_void_p, C.c_double], C.c_int),
    "dsx_lab_log": ([C.c_void_p, C.c_double, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_nccl_unique_id": ([C.c_void_p], C.c_int),
    "dsx_lab_comm_init": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int], C.c_int),
    "dsx_lab_comm_init_local": ([C.c_void_p, C.c_int, C.c_int], C.c_int),
    "dsx_lab_set_overlap": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_lab_set_pipeline": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_lab_set_noise_horizon": ([C.c_void_p, C.c_longlong], C.c_int),
    "dsx_lab_link_probe": ([C.c_void_p, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "dsx_lab_set_link": ([C.c_void_p, C.c_double, C.c_double], C.c_int),
    "dsx_lab_profile": ([C.c_void_p, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_last_timeline": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_event_record": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_lab_event_elapsed": ([C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)], C.c_int),
    "dsx_lab_set_instrument": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_lab_last_step_times": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_lab_launch_count": ([C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "dsx_mt_jump_selftest": ([C.c_ulonglong, C.POINTER(C.c_int)], C.c_int),
    "dsx_sync_plan": ([C.c_int, C.c_int, C.POINTER(C.c_int)], C.c_int),
    "dsx_p2p_average_selftest": ([C.c_int, C.c_longlong, C.POINTER(C.c_double)], C.c_int),
}


# include/dsx_nn.h: the NN local step
_NN_SIGS = {
    "dsx_gemm": ([C.POINTER(GemmDescC)], C.c_int),
    "dsx_mlp_create": ([C.POINTER(MlpDescC), C.POINTER(C.c_void_p)], C.c_int),
    "dsx_mlp_destroy": ([C.c_void_p], C.c_int),
    "dsx_mlp_param_layout": ([C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p], C.c_int),
    "dsx_mlp_set_params": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_mlp_get_params": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_mlp_get_state": ([C.c_void_p, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_mlp_set_batch": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int], C.c_int),
    "dsx_mlp_step": ([C.c_void_p, C.c_double, C.c_longlong, C.c_void_p], C.c_int),
    "dsx_mlp_last_loss": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_mlp_sync": ([C.c_void_p], C.c_int),
    "dsx_mlp_comm_init": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int),
    "dsx_mlp_set_instrument": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_mlp_last_step_times": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_mlp_profile": ([C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_mlp_event_record": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_mlp_event_elapsed": ([C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)], C.c_int),
    "dsx_mlp_launch_count": ([C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "dsx_mlp_set_graphs": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_mlp_set_link": ([C.c_void_p, C.c_double, C.c_double], C.c_int),
    "dsx_mlp_set_overlap": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_cnn_create": ([C.POINTER(CnnDescC), C.POINTER(C.c_void_p)], C.c_int),
    "dsx_cnn_destroy": ([C.c_void_p], C.c_int),
    "dsx_cnn_param_layout": ([C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p],
                             C.c_int),
    "dsx_cnn_set_params": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_cnn_get_params": ([C.c_void_p, C.c_int, C.c_void_p], C.c_int),
    "dsx_cnn_set_batch": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int], C.c_int),
    "dsx_cnn_step": ([C.c_void_p, C.c_double, C.c_longlong, C.c_void_p], C.c_int),
    "dsx_cnn_last_loss": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_cnn_sync": ([C.c_void_p], C.c_int),
    "dsx_cnn_comm_init": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int], C.c_int),
    "dsx_cnn_set_instrument": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_cnn_last_step_times": ([C.c_void_p, C.c_void_p], C.c_int),
    "dsx_cnn_event_record": ([C.c_void_p, C.c_int], C.c_int),
    "dsx_cnn_event_elapsed": ([C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)], C.c_int),
    "dsx_cnn_launch_count": ([C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "dsx_cnn_profile": ([C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "dsx_cnn_set_link": ([C.c_void_p, C.c_double, C.c_double], C.c_int),
    "dsx_cnn_set_overlap": ([C.c_void_p, C.c_int], C.c_int),
}
_SIGS.update(_NN_SIGS)


def exported_symbols(header: str = "dsx.h"):
    """Every entry point include/<header> declares (checked by the CPU tests)."""
    return sorted(_NN_SIGS) if header == "dsx_nn.h" else sorted(k for k in _SIGS if k not in _NN_SIGS)


def load_dsx():
    global _dsx
    if _dsx is None:
        if not os.path.exists(DSX_PATH):
            raise RuntimeError(
                f"{DSX_PATH} is missing: build the native engine first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make`)")
        lib = C.CDLL(DSX_PATH, mode=C.RTLD_GLOBAL)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _dsx = lib
    return _dsx


def call(name: str, *args) -> None:
    lib = load_dsx()
    status = getattr(lib, name)(*args)
    if status != DSX_OK:
        raise DsxError(status, name, lib.dsx_last_error().decode(errors="replace"))
