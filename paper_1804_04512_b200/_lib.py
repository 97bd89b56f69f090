"""ctypes binding of libb200nn.so (include/b200nn.h). No fallback: if the CUDA library cannot be
built or loaded, every entry point raises -- the product path never drops to a CPU
implementation."""
from __future__ import annotations

import ctypes as C
import os
import shutil
from pathlib import Path

from . import build as _build


class Error(RuntimeError):
    """fastnn::Error (config.hpp:11)."""


class ShapeError(Error):
    pass


class ParamError(Error):
    pass


class LabelError(Error):
    pass


class SpecError(Error):
    pass


class BoundsError(Error):
    pass


class CudaError(Error):
    pass


class NcclError(Error):
    pass


class OutOfMemory(Error):
    pass


class FormatError(Error):
    """fastnn::FormatError (config.hpp): malformed or mismatched checkpoint."""


class LengthError(Error):
    """fastnn::LengthError (config.hpp): checkpoint truncated."""


class DataMissingError(Error):
    """fastnn::DataMissingError (config.hpp): a file cannot be opened or written."""


class ConsistencyError(Error):
    """fastnn::ConsistencyError (config.hpp): mutually inconsistent inputs."""


class DataError(Error):
    """fastnn::DataError (config.hpp): unusable dataset (e.g. empty)."""


_ERRORS = {1: ShapeError, 2: ParamError, 3: LabelError, 4: CudaError, 5: NcclError, 6: OutOfMemory, 7: SpecError,
           8: BoundsError, 9: Error, 10: FormatError, 11: LengthError, 12: DataMissingError,
           13: ConsistencyError, 14: DataError}

_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_LL = C.POINTER(C.c_longlong)
_VP = C.c_void_p
_U = C.POINTER(C.c_uint)


class LayerDescC(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_", C.c_longlong), ("out", C.c_longlong), ("k", C.c_longlong),
                ("kh", C.c_longlong), ("kw", C.c_longlong), ("pad", C.c_longlong), ("p", C.c_float)]


class NetworkSpecC(C.Structure):
    _fields_ = [("input_rank", C.c_int), ("input", C.c_longlong * 3), ("layers", C.POINTER(LayerDescC)),
                ("n_layers", C.c_int), ("optimizer", C.c_int), ("lr", C.c_float), ("momentum", C.c_float),
                ("weight_decay", C.c_float), ("batch_size", C.c_longlong), ("seed", C.c_uint)]


_SIGS = {
    "b2n_last_error": ([], C.c_char_p),
    "b2n_version": ([], C.c_int),
    "b2n_device_count": ([_I], C.c_int),
    "b2n_build_network": ([C.POINTER(NetworkSpecC), C.c_int, C.c_int, C.POINTER(_VP)], C.c_int),
    "b2n_net_destroy": ([_VP], C.c_int),
    "b2n_net_num_params": ([_VP, _I], C.c_int),
    "b2n_net_param_shape": ([_VP, C.c_int, _I, _LL], C.c_int),
    "b2n_net_get_param": ([_VP, C.c_int, C.c_int, _F], C.c_int),
    "b2n_net_set_param": ([_VP, C.c_int, C.c_int, _F], C.c_int),
    "b2n_net_set_hparams": ([_VP, C.c_float, C.c_float, C.c_float], C.c_int),
    "b2n_train_minibatch": ([_VP, _F, _F, C.c_longlong, _D], C.c_int),
    "b2n_train_minibatch_labels": ([_VP, _F, _I, C.c_longlong, _D], C.c_int),
    "b2n_net_train_stream": ([_VP, _F, _I, C.c_longlong, C.c_longlong, _D], C.c_int),
    "b2n_forward_batch": ([_VP, _F, C.c_longlong, _F, _I], C.c_int),
    "b2n_net_forward_backward": ([_VP, _F, _I, C.c_longlong, C.c_longlong, _D], C.c_int),
    "b2n_net_num_layers": ([_VP, C.POINTER(C.c_longlong)], C.c_int),
    "b2n_net_layer_output": ([_VP, C.c_int, C.c_longlong, _F, C.POINTER(C.c_ubyte)], C.c_int),
    "b2n_net_apply_update": ([_VP], C.c_int),
    "b2n_net_grad_buffer": ([_VP, C.POINTER(_F), _LL], C.c_int),
    "b2n_nccl_unique_id": ([C.c_char_p], C.c_int),
    "b2n_net_dp_init": ([_VP, C.c_char_p, C.c_int, C.c_int], C.c_int),
    "b2n_net_stage": ([_VP, _F, _I, C.c_longlong], C.c_int),
    "b2n_net_run_staged": ([_VP, C.c_int, C.c_longlong], C.c_int),
    "b2n_net_loss": ([_VP, _D], C.c_int),
    "b2n_net_fit": ([_VP, _F, _I, C.c_longlong, C.c_int, _D, _D, _D], C.c_int),
    "b2n_net_evaluate": ([_VP, _F, _I, C.c_longlong, _D], C.c_int),
    "b2n_save_network": ([_VP, C.c_char_p, C.c_int], C.c_int),
    "b2n_load_network": ([_VP, C.c_char_p, C.c_int], C.c_int),
    "b2n_dbn_pretrain": ([C.POINTER(_VP), C.c_int, _F, C.c_longlong, C.c_int, C.c_float, C.c_longlong, _VP, _VP,
                          _D], C.c_int),
    "b2n_batch_order": ([C.c_longlong, C.c_uint, C.c_int, _LL], C.c_int),
    "b2n_net_stream": ([_VP, C.POINTER(_VP)], C.c_int),
    "b2n_net_kernels_per_step": ([_VP, C.c_longlong, _I], C.c_int),
    "b2n_net_profile": ([_VP, C.c_longlong, C.c_int, C.c_int, _D, C.c_char_p, C.c_int, _I], C.c_int),
    "b2n_rbm_profile": ([_VP, C.c_int, C.c_float, C.c_longlong, C.c_int, _D, C.c_char_p, C.c_int, _I], C.c_int),
    "b2n_rbm_kernels_per_step": ([_VP, _I], C.c_int),
    "b2n_rbm_create": ([C.c_longlong, C.c_longlong, C.c_int, C.c_int, C.POINTER(_VP)], C.c_int),
    "b2n_rbm_destroy": ([_VP], C.c_int),
    "b2n_rbm_init": ([_VP, C.c_uint], C.c_int),
    "b2n_rbm_set": ([_VP, _F, _F, _F], C.c_int),
    "b2n_rbm_get": ([_VP, _F, _F, _F], C.c_int),
    "b2n_cd_k_update": ([_VP, _F, C.c_longlong, C.c_int, C.c_float, _D, C.c_longlong, _D], C.c_int),
    "b2n_rbm_last_states": ([_VP, _F, _F, _F, _F], C.c_int),
    "b2n_rbm_dp_init": ([_VP, C.c_char_p, C.c_int, C.c_int], C.c_int),
    "b2n_rbm_stage": ([_VP, _F, _D, C.c_longlong], C.c_int),
    "b2n_rbm_run_staged": ([_VP, C.c_int, C.c_float, C.c_longlong], C.c_int),
    "b2n_rbm_recon": ([_VP, _D], C.c_int),
    "b2n_rbm_set_grad_only": ([_VP, C.c_int], C.c_int),
    "b2n_rbm_get_grad": ([_VP, _F, _F, _F], C.c_int),
    "b2n_rbm_set_grad": ([_VP, _F, _F, _F], C.c_int),
    "b2n_rbm_apply_update": ([_VP, C.c_float, C.c_longlong], C.c_int),
    "b2n_rbm_train_stream": ([_VP, _F, _D, C.c_longlong, C.c_longlong, C.c_float, _D], C.c_int),
    "b2n_rbm_stream": ([_VP, C.POINTER(_VP)], C.c_int),
    "b2n_op_conv_forward": ([C.c_int, _VP, _F, _F, _F, _F], C.c_int),
    "b2n_op_conv_backward": ([C.c_int, _VP, _F, _F, _F, _F, _F, _F], C.c_int),
    "b2n_op_pool_forward": ([C.c_int, C.c_int, C.c_longlong, C.c_longlong, C.c_longlong, _F, _F, _F], C.c_int),
    "b2n_op_pool_backward": ([C.c_int, C.c_int, C.c_longlong, C.c_longlong, C.c_longlong, _F, _F, _F], C.c_int),
    "b2n_op_activation_apply": ([C.c_int, C.c_int, C.c_longlong, _F, _F], C.c_int),
    "b2n_op_activation_gradient": ([C.c_int, C.c_int, C.c_longlong, _F, _F, _F], C.c_int),
    "b2n_op_softmax": ([C.c_int, C.c_longlong, C.c_longlong, _F, _F], C.c_int),
    "b2n_op_softmax_cross_entropy": ([C.c_int, C.c_longlong, C.c_longlong, _F, _F, _F, _D], C.c_int),
    "b2n_rbm_set_rng": ([_VP, _U], C.c_int),
    "b2n_rbm_get_rng": ([_VP, _U], C.c_int),
    "b2n_crbm_set_rng": ([_VP, _U], C.c_int),
    "b2n_crbm_train_stream": ([_VP, _F, _D, C.c_longlong, C.c_longlong, C.c_float, _D], C.c_int),
    "b2n_crbm_get_rng": ([_VP, _U], C.c_int),
    "b2n_mt19937_draw": ([C.c_int, _U, _D, C.c_longlong], C.c_int),
    "b2n_crbm_create": ([C.c_int] * 6 + [C.c_int, C.c_int, C.POINTER(_VP)], C.c_int),
    "b2n_crbm_destroy": ([_VP], C.c_int),
    "b2n_crbm_init": ([_VP, C.c_uint], C.c_int),
    "b2n_crbm_set": ([_VP, _F, _F, _F], C.c_int),
    "b2n_crbm_get": ([_VP, _F, _F, _F], C.c_int),
    "b2n_crbm_cd_update": ([_VP, _F, C.c_longlong, C.c_float, _D, C.c_longlong, _D], C.c_int),
    "b2n_crbm_last_states": ([_VP, _F, _F, _F, _F], C.c_int),
    "b2n_crbm_keep_states": ([_VP, C.c_int], C.c_int),
    "b2n_crbm_dp_init": ([_VP, C.c_char_p, C.c_int, C.c_int], C.c_int),
    "b2n_crbm_stage": ([_VP, _F, _D, C.c_longlong], C.c_int),
    "b2n_crbm_run_staged": ([_VP, C.c_int, C.c_float, C.c_longlong], C.c_int),
    "b2n_crbm_recon": ([_VP, _D], C.c_int),
    "b2n_crbm_kernels_per_step": ([_VP, _I], C.c_int),
    "b2n_crbm_stream": ([_VP, C.POINTER(_VP)], C.c_int),
    "b2n_crbm_profile": ([_VP, C.c_int, C.c_float, C.c_longlong, C.c_int, _D, C.c_char_p, C.c_int, _I], C.c_int),
    "b2n_gemm": ([_VP, C.c_longlong, C.c_int, _VP, C.c_longlong, C.c_int, _VP, C.c_longlong, C.c_longlong,
                  C.c_longlong, C.c_longlong, C.c_int, _VP], C.c_int),
    "b2n_sgd_momentum_step": ([_VP, _VP, _VP, C.c_longlong, C.c_float, C.c_float, C.c_float, _VP], C.c_int),
}

EXPORTED = sorted(_SIGS)

_lib: C.CDLL | None = None


def lib_path() -> Path:
    return _build.LIB


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if needed and nvcc is present) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if build_if_missing and (not path.exists() or not _build.up_to_date()):
        if shutil.which(_build.NVCC) or os.path.exists(_build.NVCC):
            _build.build()
    if not path.exists():
        raise ImportError(f"{path} is missing and could not be built; the B200 path has no CPU fallback")
    lib = C.CDLL(str(path))
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = load().b2n_last_error().decode(errors="replace")
        raise _ERRORS.get(status, Error)(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
