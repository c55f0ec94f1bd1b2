"""ctypes loader for the in-tree engine library (libppc.so, built for sm_100a).

The product path has no CPU fallback: if the library is missing or no B200 is
visible, calls raise instead of computing something else.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libppc.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "ppc.h")

_lib = None

PPC_HOST, PPC_DEVICE = 0, 1


class EngineMissing(RuntimeError):
    """libppc.so has not been built (run __graft_entry__.build())."""


def exported_symbols_from_header(path: str = HEADER) -> list[str]:
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ppc_[a-z0-9_]+)\s*\(", text)))


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineMissing(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    pd = C.POINTER(C.c_double)
    i64 = C.c_int64
    vp = C.c_void_p
    sig = {
        "ppc_last_error": (C.c_char_p, []),
        "ppc_version": (C.c_int, []),
        "ppc_device_count": (C.c_int, []),
        "ppc_set_device": (C.c_int, [C.c_int]),
        "ppc_set_stream": (C.c_int, [vp]),
        "ppc_get_stream": (vp, []),
        "ppc_synchronize": (C.c_int, []),
        "ppc_trim_workspace": (C.c_int, []),
        "ppc_launch_count": (i64, [C.c_int]),
        "ppc_timing_enable": (C.c_int, [C.c_int]),
        "ppc_set_gemm_path": (C.c_int, [C.c_int]),
        "ppc_set_ozaki": (C.c_int, [C.c_int]),
        "ppc_get_ozaki": (C.c_int, []),
        "ppc_facewise_strided": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, i64, i64]),
        "ppc_star_inverse": (C.c_int, [vp, i64, i64, vp, i64, C.c_double, vp]),
        "ppc_reshard_slices": (C.c_int, [vp, i64, i64, i64, i64, vp]),
        "ppc_sym_eig_split_begin": (C.c_int, [vp, i64, i64, C.POINTER(C.c_int64)]),
        "ppc_sym_eig_split_vectors": (C.c_int, [i64, i64, i64, vp]),
        "ppc_sym_eig_split_finish": (C.c_int, [i64, vp, i64, i64, vp]),
        "ppc_sym_eig_split_release": (C.c_int, [i64]),
        "ppc_ozaki_syrk_batched": (C.c_int, [vp, i64, i64, i64, i64, i64, vp]),
        "ppc_timing_report": (C.c_int, [C.c_char_p, i64, C.c_int]),
        "ppc_mode3_product": (C.c_int, [vp, i64, i64, i64, vp, i64, C.c_int, vp, C.c_int]),
        "ppc_mode_product": (C.c_int, [vp, i64, i64, i64, vp, i64, C.c_int, vp, C.c_int]),
        "ppc_facewise_product": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, C.c_int]),
        "ppc_frobenius_norm": (C.c_int, [vp, i64, pd, C.c_int]),
        "ppc_svd_batched": (C.c_int, [vp, i64, i64, i64, i64, vp, vp, vp, C.c_int]),
        "ppc_data_dependent_q": (C.c_int, [vp, i64, i64, i64, i64, vp, vp, C.POINTER(C.c_int), C.c_int]),
        "ppc_projection_error": (C.c_int, [vp, i64, i64, i64, vp, i64, pd, C.c_int]),
        "ppc_dct_q": (C.c_int, [i64, i64, vp]),
        "ppc_haar_q": (C.c_int, [i64, i64, vp]),
        "ppc_random_orthogonal_q": (C.c_int, [i64, i64, C.c_uint64, vp]),
        "ppc_identity_q": (C.c_int, [i64, i64, vp]),
        "ppc_check_stiefel": (C.c_int, [vp, i64, i64]),
        "ppc_orthonormalize": (C.c_int, [vp, i64, i64, vp]),
        "ppc_star_q_product": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, i64, C.c_double, vp, C.c_int]),
        "ppc_tsvdq": (C.c_int, [vp, i64, i64, i64, vp, i64, i64, vp, vp, vp, C.c_int]),
        "ppc_tsvdq_reconstruct": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, i64, i64, vp, C.c_int]),
        "ppc_tsvdq_error": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, i64, i64, pd, pd, pd, C.c_int]),
        "ppc_relative_error": (C.c_int, [vp, vp, i64, pd, C.c_int]),
        "ppc_tsvdq_relative_error": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, i64, i64, pd, C.c_int]),
        "ppc_gram_plan": (C.c_int, [i64, i64, C.POINTER(i64), C.POINTER(i64)]),
        "ppc_gram_partials": (C.c_int, [vp, i64, i64, i64, i64, i64, vp, C.c_int]),
        "ppc_tree_reduce": (C.c_int, [vp, i64, i64, C.c_int]),
        "ppc_sym_eig_top": (C.c_int, [vp, i64, i64, vp, vp, C.c_int]),
        "ppc_gram_partials_keep": (C.c_int, [vp, i64, i64, i64, i64, i64, vp, C.POINTER(C.c_int64),
                                            C.POINTER(C.c_int)]),
        "ppc_mode3_forward_digits": (C.c_int, [i64, vp, i64, vp]),
        "ppc_digits_release": (C.c_int, [i64]),
        "ppc_slice_residual_sums": (C.c_int, [vp, i64, i64, i64, i64, vp, vp, vp, pd, C.c_int]),
        "ppc_gram_trace": (C.c_int, [vp, i64, pd, C.c_int]),
        "ppc_recon_residual_block": (C.c_int, [vp, i64, i64, i64, i64, vp, vp, vp, i64, i64, vp, i64, i64, pd, C.c_int]),
        "ppc_tsvdq2": (C.c_int, [vp, i64, i64, i64, vp, i64, C.c_double, vp, vp, vp, C.POINTER(i64), C.c_int]),
        "ppc_tsvdq2_reconstruct": (C.c_int, [vp, vp, vp, vp, i64, i64, i64, i64, C.POINTER(i64), vp, C.c_int]),
        "ppc_tsvdq2_error": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, i64, C.POINTER(i64), pd, pd, pd, C.c_int]),
        "ppc_gemm_strided": (C.c_int, [i64, i64, i64, i64, C.c_double, vp, i64, i64, C.c_int, vp, i64, i64,
                                       C.c_int, vp, i64, i64]),
        "ppc_pt3_info": (C.c_int, [C.c_char_p, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
        "ppc_pt3_read": (C.c_int, [C.c_char_p, vp, i64, C.c_int]),
        "ppc_pt3_write": (C.c_int, [C.c_char_p, vp, i64, i64, i64, C.c_int]),
        "ppc_star_m_product": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, vp, C.c_int]),
        "ppc_hosvd": (C.c_int, [vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp, C.c_int]),
        "ppc_hosvd_reconstruct": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, C.c_int]),
        "ppc_matrix_svd_baseline": (C.c_int, [vp, i64, i64, i64, i64, vp, vp, vp, pd, C.c_int]),
        "ppc_tsvdq_sweep": (C.c_int, [vp, i64, i64, i64, C.POINTER(i64), i64, C.POINTER(i64), i64, vp, vp, C.c_int]),
        "ppc_tsvdq_compress": (C.c_int, [vp, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, pd, C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
