"""ctypes binding of libdapple.so (include/dapple.h).

The library is built in-tree by ``paper_2007_01045_b200/build.py``; there is
no fallback: if it is missing, importing the product fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdapple.so")

_lib = None


class DappleError(RuntimeError):
    pass


class GemmDesc(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int), ("batch", ctypes.c_int),
        ("A", ctypes.c_void_p), ("lda", ctypes.c_longlong), ("a_batch_stride", ctypes.c_longlong),
        ("a_mn_major", ctypes.c_int),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_longlong), ("b_batch_stride", ctypes.c_longlong),
        ("b_mn_major", ctypes.c_int),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_longlong), ("zdiv", ctypes.c_int),
        ("s_zo", ctypes.c_longlong), ("s_zi", ctypes.c_longlong), ("ndiv", ctypes.c_int),
        ("s_no", ctypes.c_longlong), ("epi", ctypes.c_uint32), ("alpha", ctypes.c_float),
        ("bias", ctypes.c_void_p), ("aux_in", ctypes.c_void_p), ("resid", ctypes.c_void_p),
        ("aux_out", ctypes.c_void_p), ("force_bn", ctypes.c_int), ("force_1sm", ctypes.c_int),
        ("trace", ctypes.c_void_p), ("colsum", ctypes.c_void_p),
        ("conv_x", ctypes.c_void_p), ("conv_operand", ctypes.c_int), ("conv_n", ctypes.c_int),
        ("conv_h", ctypes.c_int), ("conv_w", ctypes.c_int), ("conv_c", ctypes.c_int),
        ("split_ws", ctypes.c_void_p), ("split_ws_bytes", ctypes.c_size_t),
    ]


EPI_OUT_BF16, EPI_OUT_F32, EPI_OUT_F32_ACC = 0, 1, 2
EPI_BIAS, EPI_GELU, EPI_RELU, EPI_AUX_OUT = 1 << 2, 1 << 3, 1 << 4, 1 << 5
EPI_DGELU, EPI_DRELU, EPI_RESID = 1 << 6, 1 << 7, 1 << 8
EPI_COLSUM = 1 << 9

_VP, _I, _LL, _F, _U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_float, ctypes.c_uint64

_PROTOS = {
    "dpl_host_call": (ctypes.c_char_p, [ctypes.c_char_p]),
    "dpl_last_error": (ctypes.c_char_p, []),
    "dpl_version": (ctypes.c_char_p, []),
    "dpl_k_gemm": (_I, [ctypes.POINTER(GemmDesc), _VP]),
    "dpl_k_attention_fwd": (_I, [_VP, _VP, _LL, _VP, _I, _I, _I, _I, _VP]),
    "dpl_k_attention_fwd_traced": (_I, [_VP, _VP, _LL, _VP, _I, _I, _I, _I, _VP, _VP]),
    "dpl_k_attention_bwd": (_I, [_VP, _VP, _LL, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _I, _VP]),
    "dpl_k_attention_bwd_traced": (_I, [_VP, _VP, _LL, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _I, _VP, _VP]),
    "dpl_k_layernorm_fwd": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _F, _VP]),
    "dpl_k_layernorm_bwd": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _VP]),
    "dpl_k_layernorm_bwd_colsum": (_I, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _I, _I, _VP]),
    "dpl_k_softmax_fwd": (_I, [_VP, _VP, _I, _I, _I, _I, _VP]),
    "dpl_k_softmax_bwd": (_I, [_VP, _VP, _VP, _I, _I, _VP]),
    "dpl_k_colsum_acc": (_I, [_VP, _VP, _I, _I, _VP]),
    "dpl_k_mse_loss": (_I, [_VP, _VP, _VP, _VP, _LL, _F, _VP]),
    "dpl_k_sgd_apply": (_I, [_VP, _VP, _VP, _LL, _F, _VP]),
    "dpl_k_fill_tokens": (_I, [_VP, _LL, _U64, _U64, _LL, _I, _VP]),
    "dpl_k_embed_fwd": (_I, [_VP, _VP, _VP, _VP, _I, _I, _I, _VP]),
    "dpl_k_embed_bwd": (_I, [_VP, _VP, _VP, _VP, _I, _I, _I, _VP]),
    "dpl_k_cross_entropy": (_I, [_VP, _VP, _VP, _I, _I, _F, _VP]),
    "dpl_k_cross_entropy_padded": (_I, [_VP, _VP, _VP, _I, _I, _I, _F, _VP]),
    "dpl_k_im2col3x3": (_I, [_VP, _VP, _I, _I, _I, _I, _I, _VP]),
    "dpl_k_col2im3x3": (_I, [_VP, _VP, _I, _I, _I, _I, _I, _VP]),
    "dpl_k_maxpool2_fwd": (_I, [_VP, _VP, _I, _I, _I, _I, _VP]),
    "dpl_k_maxpool2_relu_bwd": (_I, [_VP, _VP, _VP, _I, _I, _I, _I, _VP]),
    "dpl_k_relu_bwd": (_I, [_VP, _VP, _VP, _LL, _VP]),
    "dpl_k_fill_uniform_bf16": (_I, [_VP, _LL, _U64, _U64, _LL, _F, _VP]),
    "dpl_k_fill_uniform_f32": (_I, [_VP, _LL, _U64, _U64, _LL, _F, _VP]),
    "dpl_k_launch_count": (_LL, []),
    "dpl_exec_create": (_I, [ctypes.c_char_p, _I, ctypes.POINTER(_VP)]),
    "dpl_exec_export": (_I, [_VP, _VP, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "dpl_exec_connect": (_I, [_VP, _VP, ctypes.c_size_t, _I]),
    "dpl_exec_nccl_id": (_I, [_VP]),
    "dpl_exec_nccl_init": (_I, [_VP, _VP]),
    "dpl_exec_step": (_I, [_VP, _VP, _VP, ctypes.POINTER(_F)]),
    "dpl_exec_step_launch": (_I, [_VP, _VP, _VP]),
    "dpl_exec_step_finish": (_I, [_VP, ctypes.POINTER(_F)]),
    "dpl_exec_prepare": (_I, [_VP]),
    "dpl_exec_timeline": (ctypes.c_char_p, [_VP]),
    "dpl_exec_read_tensor": (_I, [_VP, ctypes.c_char_p, _I, _VP, ctypes.c_size_t]),
    "dpl_exec_info": (_I, [_VP, ctypes.c_char_p, ctypes.c_size_t]),
    "dpl_exec_read_probe": (_I, [_VP, _I, ctypes.c_char_p, _VP, ctypes.c_size_t]),
    "dpl_exec_clock_calibrate": (_I, [_VP, _I, ctypes.POINTER(_LL)]),
    "dpl_exec_gemm_profile": (_I, [_VP, _I]),
    "dpl_exec_gemm_profile_json": (ctypes.c_char_p, [_VP]),
    "dpl_exec_layer_profile": (ctypes.c_char_p, [_VP, ctypes.c_int]),
    "dpl_exec_disconnect": (_I, [_VP]),
    "dpl_exec_destroy": (None, [_VP]),
}


def _preload_torch_nccl():
    """libdapple needs libnccl.so.2; make it resolve to the copy torch bundles
    (nvidia/nccl), so loading libdapple before `import torch` cannot pin the
    older system NCCL that libtorch_cuda then fails to link against."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for root in (spec.submodule_search_locations or []) if spec else []:
        path = os.path.join(root, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(path):
            ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
            return


def lib():
    """Loads libdapple.so (building it first if this is a source checkout)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DappleError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    _preload_torch_nccl()
    handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(handle, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


def exported_symbols():
    return list(_PROTOS)


def check(rc: int):
    if rc != 0:
        raise DappleError(lib().dpl_last_error().decode())
