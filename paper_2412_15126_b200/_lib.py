"""ctypes binding of libslotrank_b200.so (the C-ABI in include/slotrank_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2412_15126_b200.build``).  There is no fallback: if the
shared object is missing or no CUDA device is visible, every engine
constructor raises ``RuntimeError`` naming the problem.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_int, c_longlong, c_size_t, c_uint64, c_void_p, POINTER

__all__ = ["lib", "LIB_PATH", "check", "SrkError", "EXPORTS"]

LIB_PATH = os.environ.get("SRK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     "libslotrank_b200.so")

_u64p = c_void_p  # device or host pointers passed as integers

# name -> argtypes (all return int unless listed in _RESTYPES)
EXPORTS = {
    "srk_last_error": [],
    "srk_version": [],
    "srk_kernel_launches": [],
    "srk_fp64_probe": [c_int, c_int, c_void_p, c_void_p],
    "srk_ctx_create": [c_int, c_int, POINTER(c_uint64), POINTER(c_uint64), c_int, c_int, c_int,
                       POINTER(c_void_p)],
    "srk_ctx_destroy": [c_void_p],
    "srk_workspace_bytes": [c_void_p],
    "srk_ctx_set_branch_stream": [c_void_p, c_void_p],
    "srk_ntt": [c_void_p, _u64p, c_int, c_longlong, c_int, c_int, c_int, c_void_p],
    "srk_ntt_ext": [c_void_p, _u64p, c_int, c_longlong, c_int, c_int, c_void_p],
    "srk_addsub": [c_void_p, _u64p, _u64p, _u64p, c_int, c_int, c_void_p],
    "srk_add_const": [c_void_p, _u64p, POINTER(c_uint64), _u64p, c_int, c_void_p],
    "srk_add_plain": [c_void_p, _u64p, _u64p, _u64p, c_int, c_void_p],
    "srk_mul_const": [c_void_p, _u64p, c_int, POINTER(c_uint64), _u64p, c_int, c_void_p],
    "srk_mul_plain": [c_void_p, _u64p, _u64p, _u64p, c_int, c_void_p],
    "srk_tensor": [c_void_p, _u64p, _u64p, _u64p, c_int, c_void_p],
    "srk_rescale": [c_void_p, _u64p, _u64p, c_int, c_void_p, c_void_p],
    "srk_mul_const_rescale": [c_void_p, _u64p, c_int, POINTER(c_uint64), _u64p, c_int, c_void_p,
                              c_void_p],
    "srk_mul_plain_rescale": [c_void_p, _u64p, _u64p, _u64p, c_int, c_void_p, c_void_p],
    "srk_keyswitch": [c_void_p, _u64p, _u64p, _u64p, _u64p, c_int, c_void_p, c_void_p],
    "srk_mul_relin": [c_void_p, _u64p, _u64p, _u64p, _u64p, c_int, c_void_p, c_void_p],
    "srk_mul_relin_rescale": [c_void_p, _u64p, _u64p, _u64p, _u64p, c_int, c_void_p, c_void_p],
    "srk_automorph": [c_void_p, _u64p, _u64p, c_longlong, c_uint64, c_void_p],
    "srk_rotate": [c_void_p, _u64p, _u64p, _u64p, c_int, c_uint64, c_void_p, c_void_p],
    "srk_rescale_batch": [c_void_p, _u64p, c_longlong, _u64p, c_longlong, c_int, c_int, c_void_p,
                          c_void_p],
    "srk_mul_relin_batch": [c_void_p, _u64p, _u64p, c_longlong, _u64p, _u64p, c_longlong, c_int,
                            c_int, c_int, c_void_p, c_void_p],
    "srk_mul_relin_ptrs": [c_void_p, c_void_p, c_void_p, c_int, _u64p, _u64p, c_longlong, c_int, c_int,
                           c_void_p, c_void_p],
    "srk_addsub_batch": [c_void_p, _u64p, _u64p, _u64p, c_int, c_int, c_int, c_void_p],
    "srk_add_plain_batch": [c_void_p, _u64p, _u64p, c_longlong, POINTER(c_uint64), _u64p, c_int,
                            c_int, c_void_p],
    "srk_mul_const_rescale_batch": [c_void_p, _u64p, c_longlong, c_int, POINTER(c_uint64), _u64p,
                                    c_int, c_int, c_void_p, c_void_p],
    "srk_mul_plain_rescale_batch": [c_void_p, _u64p, _u64p, c_longlong, _u64p, c_int, c_int,
                                    c_void_p, c_void_p],
    "srk_rotate_batch": [c_void_p, _u64p, c_longlong, _u64p, _u64p, c_longlong, c_int, c_int,
                         c_uint64, c_void_p, c_void_p],
    "srk_rotate_hoisted": [c_void_p, _u64p, c_longlong, c_int, c_int, POINTER(c_void_p),
                           POINTER(c_uint64), POINTER(c_void_p), c_longlong, c_int, c_void_p,
                           c_void_p],
    "srk_uniform": [c_void_p, _u64p, c_int, c_int, c_uint64, c_uint64, c_void_p],
    "srk_small_to_ntt": [c_void_p, _u64p, _u64p, c_int, c_int, c_void_p],
    "srk_square": [c_void_p, _u64p, _u64p, c_int, c_void_p],
    "srk_keygen": [c_void_p, _u64p, _u64p, _u64p, c_uint64, c_uint64, _u64p, c_void_p, c_void_p],
    "srk_keygen_galois": [c_void_p, _u64p, _u64p, c_uint64, c_uint64, c_uint64, _u64p, c_void_p,
                          c_void_p],
    "srk_permute_key": [c_void_p, _u64p, c_uint64, c_void_p, c_void_p],
    "srk_encrypt": [c_void_p, _u64p, _u64p, _u64p, c_uint64, c_uint64, _u64p, c_int, c_void_p,
                    c_void_p],
    "srk_decrypt_limb0": [c_void_p, _u64p, _u64p, _u64p, c_int, c_void_p, c_void_p],
    "srk_lincomb": [c_void_p, POINTER(c_void_p), POINTER(c_int), c_int, _u64p, _u64p, c_int, c_int,
                    c_void_p],
    "srk_lincomb_multi": [c_void_p, POINTER(c_void_p), POINTER(c_int), c_int, _u64p, _u64p, POINTER(c_void_p),
                          c_int, c_int, c_int, c_void_p],
    "srk_reduce_mod": [c_void_p, _u64p, c_int, c_int, c_void_p],
    "srk_encode_plain": [c_void_p, _u64p, _u64p, c_int, c_void_p],
}
_RESTYPES = {"srk_last_error": ctypes.c_char_p, "srk_workspace_bytes": c_size_t,
             "srk_kernel_launches": ctypes.c_ulonglong}


class SrkError(RuntimeError):
    pass


_lib = None


def lib():
    """Load (once) and return the CUDA library; raise if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, argtypes in EXPORTS.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, c_int)
        _lib = handle
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().srk_last_error().decode(errors="replace")
        raise SrkError(f"libslotrank_b200 error {rc}: {msg}")
