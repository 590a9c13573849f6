"""Thin ctypes binding of the C ABI in include/pa.h (argument marshalling only).

Every step of the hash runs in the CUDA kernels of ``_pa.so``; this module only
converts Python/torch arguments to pointers and sizes.  There is no CPU fallback:
if the shared library is missing, importing this module raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PA_DEV_LIB: an in-tree A/B build of the same sources (scripts/build_variant.sh), development only
LIB_PATH = os.environ.get("PA_DEV_LIB") or os.path.join(_HERE, "_pa.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc -gencode arch=compute_100a,code=sm_100a); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

PA_OK = 0
PA_E_PARAM = -1
PA_E_INSUFFICIENT_INPUT = -2
PA_E_BOUND = -3
PA_E_NOMEM = -4
PA_E_CUDA = -5
PA_E_STATE = -6
PA_E_NCCL = -7
_CODES = {0: "PA_OK", -1: "PA_E_PARAM", -2: "PA_E_INSUFFICIENT_INPUT", -3: "PA_E_BOUND",
          -4: "PA_E_NOMEM", -5: "PA_E_CUDA", -6: "PA_E_STATE", -7: "PA_E_NCCL"}

u64, u32, i32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_void_p


class pa_stage_plan(ctypes.Structure):
    _fields_ = [("limb_bits", u32), ("nprimes", u32), ("log2_len", u32), ("n_col", u32), ("n_row", u32),
                ("primes", u32 * 16), ("bound_log2", ctypes.c_double), ("modulus_log2", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {"limb_bits": self.limb_bits, "nprimes": self.nprimes, "log2_len": self.log2_len,
                "n_col": self.n_col, "n_row": self.n_row, "primes": list(self.primes)[: self.nprimes],
                "bound_log2": self.bound_log2, "modulus_log2": self.modulus_log2}


class pa_info(ctypes.Structure):
    _fields_ = [("n", u64), ("r", u64), ("m", u64), ("gamma", u64), ("alpha", u64), ("k", u64),
                ("block_begin", u64), ("block_end", u64), ("mmh", pa_stage_plan), ("mh", pa_stage_plan),
                ("device_bytes", u64), ("kernels_per_hash", u32), ("launches_total", u32),
                ("insecure_length", u32), ("world", i32), ("rank", i32), ("acc_words", u64),
                ("graph_captures", u32), ("graph_updates", u32), ("graph_instantiations", u32),
                ("tz_group_blocks", u32), ("p2p", u32)]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("mmh", "mh")}
        d["mmh"] = self.mmh.as_dict()
        d["mh"] = self.mh.as_dict()
        return d


# device allocator callbacks of pa_params (void *alloc(size_t, void *stream, void *user);
# void free(void *, size_t, void *stream, void *user))
DEV_ALLOC = ctypes.CFUNCTYPE(vp, ctypes.c_size_t, vp, vp)
DEV_FREE = ctypes.CFUNCTYPE(None, vp, ctypes.c_size_t, vp, vp)


class pa_params(ctypes.Structure):
    _fields_ = [("n", u64), ("r", u64), ("m", u64), ("gamma", u64), ("seed", u64),
                ("block_begin", u64), ("block_end", u64),
                ("a_words", vp), ("b_words", vp), ("c_words", vp),
                ("stream", vp), ("limb_bits", i32), ("strict", i32), ("paper_k", u64), ("mh_only", u64),
                ("toeplitz", u64), ("world", i32), ("rank", i32), ("nccl_id", ctypes.c_uint8 * 128),
                ("dev_alloc", DEV_ALLOC), ("dev_free", DEV_FREE), ("alloc_user", vp),
                ("tz_group_blocks", u64), ("p2p", i32)]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


pa_ctx_create = _sig("pa_ctx_create", vp, u64, u64, u64, u64, u64)
pa_ctx_create_ex = _sig("pa_ctx_create_ex", i32, ctypes.POINTER(pa_params), ctypes.POINTER(vp))
pa_hash = _sig("pa_hash", i32, vp, vp, vp)
pa_hash_host = _sig("pa_hash_host", i32, vp, vp, vp)
pa_hash_batch = _sig("pa_hash_batch", i32, vp, ctypes.POINTER(vp), ctypes.POINTER(vp), u32)
pa_hash_host_batch = _sig("pa_hash_host_batch", i32, vp, ctypes.POINTER(vp), ctypes.POINTER(vp), u32)
pa_mmh_partial = _sig("pa_mmh_partial", i32, vp, vp, vp)
pa_mh_merge = _sig("pa_mh_merge", i32, vp, vp, u32, vp)
pa_mmh_acc = _sig("pa_mmh_acc", i32, vp, vp, vp)
pa_tail_merge = _sig("pa_tail_merge", i32, vp, vp, u32, vp)
pa_nccl_unique_id = _sig("pa_nccl_unique_id", i32, vp)
pa_debug_build = _sig("pa_debug_build", i32)
pa_debug_selftest = _sig("pa_debug_selftest", i32)
pa_ctx_destroy = _sig("pa_ctx_destroy", None, vp)
pa_ctx_status = _sig("pa_ctx_status", i32, vp)
pa_ctx_paper_stats = _sig("pa_ctx_paper_stats", i32, vp, ctypes.POINTER(u64), ctypes.POINTER(u64))
pa_ctx_rekey = _sig("pa_ctx_rekey", i32, vp, u64)
pa_ctx_query = _sig("pa_ctx_query", i32, vp, ctypes.POINTER(pa_info))
pa_ctx_set_stream = _sig("pa_ctx_set_stream", i32, vp, vp)
pa_ctx_set_profiling = _sig("pa_ctx_set_profiling", i32, vp, i32)
pa_ctx_stage_times = _sig("pa_ctx_stage_times", i32, vp, ctypes.POINTER(ctypes.c_char_p),
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u32), i32)
pa_plan = _sig("pa_plan", i32, ctypes.POINTER(pa_params), ctypes.POINTER(pa_info))
pa_philox4x64_10 = _sig("pa_philox4x64_10", i32, u64, u64, u64, vp)
pa_expand_a = _sig("pa_expand_a", i32, u64, u64, u64, vp)
pa_expand_bc = _sig("pa_expand_bc", i32, u64, u64, vp, vp)
pa_last_error = _sig("pa_last_error", i32, ctypes.c_char_p, ctypes.c_size_t)
pa_abi_sizes = _sig("pa_abi_sizes", i32, ctypes.POINTER(u64), ctypes.POINTER(u64))
pa_derive_security_coefficient = _sig("pa_derive_security_coefficient", i32, ctypes.c_double, ctypes.POINTER(u64))
pa_select_block_count = _sig("pa_select_block_count", i32, ctypes.c_double, ctypes.POINTER(u64))
pa_select_gamma = _sig("pa_select_gamma", i32, u64, u64, ctypes.POINTER(u64), ctypes.POINTER(i32))
pa_derive_paper_params = _sig("pa_derive_paper_params", i32, u64, ctypes.c_double, u64, ctypes.c_double,
                              *([ctypes.POINTER(u64)] * 5))

EXPORTED = ["pa_ctx_create", "pa_ctx_create_ex", "pa_hash", "pa_hash_host", "pa_hash_batch", "pa_hash_host_batch", "pa_mmh_partial", "pa_mh_merge",
            "pa_ctx_destroy", "pa_ctx_status", "pa_ctx_rekey", "pa_ctx_query", "pa_ctx_set_stream", "pa_ctx_set_profiling",
            "pa_ctx_stage_times", "pa_plan", "pa_philox4x64_10", "pa_expand_a", "pa_expand_bc",
            "pa_last_error", "pa_ctx_paper_stats", "pa_derive_security_coefficient", "pa_select_block_count", "pa_select_gamma",
            "pa_derive_paper_params", "pa_mmh_acc", "pa_tail_merge", "pa_nccl_unique_id", "pa_debug_build",
            "pa_debug_selftest", "pa_abi_sizes"]


class PAError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


def last_error() -> tuple[int, str]:
    buf = ctypes.create_string_buffer(512)
    code = pa_last_error(buf, 512)
    return code, buf.value.decode(errors="replace")


def check(rc: int) -> None:
    if rc != PA_OK:
        code, msg = last_error()
        raise PAError(rc, msg)
