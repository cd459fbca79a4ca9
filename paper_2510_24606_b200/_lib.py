"""ctypes binding of libdhsa_b200.so (the C ABI declared in include/dhsa_b200.h).

The library is built in-tree by ``paper_2510_24606_b200.build``.  There is
no fallback: if the library is missing or no CUDA device is present, every
GPU entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DHSA_LIB_PATH") or os.path.join(_HERE, "libdhsa_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "dhsa_b200.h")

F64, F32, BF16 = 0, 1, 2
AGG = {"none": 0, "max": 1, "mean": 2}

i32p = C.c_void_p  # device pointers are passed as integers
vp = C.c_void_p


class Layout(C.Structure):
    _fields_ = [
        ("bounds", vp),
        ("bounds_stride", C.c_int64),
        ("nchunks", vp),
        ("plen", vp),
        ("block", C.c_int32),
        ("max_chunks", C.c_int32),
    ]


class PrefillChunks(C.Structure):
    """dhsa_prefill_chunks"""

    _fields_ = [
        ("bounds", vp),
        ("bounds_stride", C.c_int64),
        ("nchunks", vp),
        ("qtiles", vp),
        ("tiles_per_unit", C.c_int32),
    ]


PChunks = C.POINTER(PrefillChunks)


class ShardSpec(C.Structure):
    """dhsa_split_shard"""
    _fields_ = [("chunk_offset", C.c_int32), ("total_chunks", C.c_int32),
                ("total_prompt", C.c_int32), ("owns_tail", C.c_int32)]


_SIGS = {
    "dhsa_last_error": (C.c_char_p, []),
    "dhsa_version": (C.c_int, []),
    "dhsa_centroids": (C.c_int, [C.c_int, vp, C.c_int64, C.c_int, C.c_int, Layout, C.c_int, vp,
                                 C.c_int64, vp]),
    "dhsa_decode_score": (C.c_int, [C.c_int, vp, vp, C.c_int64, vp, vp, vp, vp, vp, vp, C.c_int64,
                                    Layout, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int64, vp]),
    "dhsa_decode_select": (C.c_int, [vp, C.c_int64, Layout, vp, C.c_int, C.c_int, C.c_int64,
                                     C.c_int, vp, C.c_int64, vp, vp, vp]),
    "dhsa_select_scratch_size": (C.c_int64, [C.c_int]),
    "dhsa_attn_workspace_size": (C.c_int64, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    "dhsa_attn": (C.c_int, [C.c_int, vp, vp, vp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                            C.c_int, vp, C.c_int64, vp, C.c_int, vp, vp, vp, vp, vp]),
    "dhsa_decode_advance": (C.c_int, [vp, C.c_int, vp]),
    "dhsa_chunk_scores": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64,
                                    C.c_int64, vp, C.c_int64, vp]),
    "dhsa_rows_select": (C.c_int, [vp, C.c_int64, vp, C.c_int, vp, C.c_int, C.c_int64, C.c_int,
                                   vp, C.c_int64, vp, vp, vp]),
    "dhsa_upsample": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp]),
    "dhsa_softmax_rows": (C.c_int, [vp, C.c_int, C.c_int64, vp, vp]),
    "dhsa_causal_probs": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp]),
    "dhsa_mask_recall": (C.c_int, [vp, C.c_int64, C.c_int, vp, vp, vp, vp]),
    "dhsa_row_cosine": (C.c_int, [vp, vp, C.c_int64, C.c_int, vp, vp]),
    "dhsa_mean": (C.c_int, [vp, C.c_int64, vp, vp]),
    "dhsa_stack_reduce": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int, vp, vp]),
    "dhsa_sketch_build": (C.c_int, [vp, C.c_int64, C.c_int, C.c_int, Layout, vp, C.c_int64, vp,
                                    vp]),
    "dhsa_sketch_select_scratch_size": (C.c_int64, [C.c_int]),
    "dhsa_decode_step_bf16": (C.c_int, [vp, vp, C.c_int64, vp, vp, C.c_int64, vp, vp, vp, vp,
                                        vp, vp, C.c_int64, Layout, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int64, C.c_int, vp, C.c_int64, vp, vp,
                                        C.c_int64, vp, vp, C.c_int, vp, vp]),
    "dhsa_decode_candidates_bf16": (C.c_int, [vp, vp, C.c_int64, vp, vp, C.c_int64, vp, vp, vp,
                                              vp, vp, vp, C.c_int64, Layout, C.c_int, C.c_int,
                                              C.c_int, C.c_int, C.c_int64, ShardSpec, vp,
                                              C.c_int64, C.c_int, vp, C.c_int64, vp, vp, vp]),
    "dhsa_split_select": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                    vp, vp, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, vp,
                                    C.c_int64, vp, C.c_int, vp]),
    "dhsa_attn_partials": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                     C.c_int, vp, C.c_int64, vp, C.c_int, vp, vp, vp, vp]),
    "dhsa_merge_partials": (C.c_int, [vp, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, vp, vp]),
    "dhsa_prefill_scores": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                                      vp]),
    "dhsa_prefill_plan_capacity": (C.c_int, [C.c_int64, C.c_int]),
    "dhsa_prefill_mask_bitsets": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.c_int, C.c_int64, PChunks, vp, vp]),
    "dhsa_prefill_plan": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int64, PChunks, C.c_int, vp, vp, vp]),
    "dhsa_prefill_attn": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int64, C.c_int, PChunks, vp, vp, C.c_int, vp, vp,
                                    vp, vp]),
    "dhsa_row_quality": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int, vp, vp, vp]),
    "dhsa_predictor_workspace_size": (C.c_int64, [C.c_int, C.c_int, C.c_int, C.c_int]),
    "dhsa_predictor_forward": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp,
                                         vp, vp, vp, C.c_double, vp, vp, vp]),
    "dhsa_attn_stream_workspace_size": (C.c_int64, [C.c_int, C.c_int, C.c_int]),
    "dhsa_attn_stream_counters": (C.c_int, [C.c_int]),
    "dhsa_attn_stream": (C.c_int, [vp, vp, vp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                                   C.c_int, vp, C.c_int64, vp, C.c_int, vp, vp, vp, vp, vp, vp]),
}

_lib = None


def header_symbols():
    """Function names declared in include/dhsa_b200.h."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(dhsa_\w+)\(", text, re.M)))


def load():
    """Load (once) and return the ctypes library handle; raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libdhsa_b200.so not found at {LIB_PATH}; build it with "
            "`python -m paper_2510_24606_b200.build` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class DhsaError(RuntimeError):
    pass


def check(rc: int):
    if rc != 0:
        msg = load().dhsa_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise DhsaError(f"libdhsa_b200 error {rc}: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2510_24606_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    load()


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def layout(bounds=None, plen=None, nchunks=None, block=0, max_chunks=0, bounds_stride=0):
    return Layout(ptr(bounds), int(bounds_stride), ptr(nchunks), ptr(plen), int(block),
                  int(max_chunks))
