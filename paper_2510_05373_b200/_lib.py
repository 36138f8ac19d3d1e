"""ctypes binding of libkvlinc.so (the C ABI declared in include/kvlinc.h).

The shared library is built in-tree (`make`, or `__graft_entry__.build()`)
and is the only compute path: there is no CPU fallback.  Importing this
module without the library, or calling a compute entry point on a host
without an sm_100 GPU, raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import c_double, POINTER, c_int, c_int32, c_int64, c_size_t, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KVLC_LIB") or os.path.join(_HERE, "libkvlinc.so")  # KVLC_LIB: tracing build

KVLC_OK, KVLC_EINVAL, KVLC_ECUDA, KVLC_ENODEV, KVLC_ENOSPC = 0, 1, 2, 3, 4
AXIS_TOKEN, AXIS_CHANNEL = 0, 1
PLACE_PRE, PLACE_POST = 0, 1
D, G, R, RANK, SLOTS = 128, 128, 128, 256, 256


class KvlcCache(ctypes.Structure):
    """Mirror of `kvlc_cache` (include/kvlinc.h)."""
    _fields_ = [("B", c_int32), ("Hkv", c_int32), ("Hq", c_int32), ("max_chunks", c_int32),
                ("kcodes", c_void_p), ("vcodes", c_void_p), ("kscale", c_void_p),
                ("kzero", c_void_p), ("vscale", c_void_p), ("vzero", c_void_p),
                ("kres", c_void_p), ("vres", c_void_p), ("S", c_void_p), ("P", c_void_p),
                ("n_chunks", c_void_p), ("res_start", c_void_p), ("res_len", c_void_p)]


class KvlcAdapter(ctypes.Structure):
    """Mirror of `kvlc_adapter`."""
    _fields_ = [("w1q", c_void_p), ("w2q", c_void_p), ("w1k", c_void_p), ("w2k", c_void_p),
                ("enabled", c_int32)]


class KvlcDecodeOpts(ctypes.Structure):
    """Mirror of `kvlc_decode_opts`."""
    _fields_ = [("chunks_per_split", c_int32), ("literal", c_int32), ("max_chunks_hint", c_int32),
                ("out_fp32", c_int32), ("ev_begin", c_void_p), ("ev_end", c_void_p)]


class KvlcError(RuntimeError):
    """A CUDA / device failure inside libkvlinc."""


_SIGS = {
    "kvlc_version": (c_int, []),
    "kvlc_last_error": (ctypes.c_char_p, []),
    "kvlc_device_ok": (c_int, []),
    "kvlc_note_cache_write": (None, [POINTER(KvlcCache)]),
    "kvlc_adapter_grads_workspace": (c_size_t, [c_int64, c_int, c_int, c_int]),
    "kvlc_adapter_grads": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p, c_int,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "kvlc_adam_step": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_double, c_double, c_double,
                               c_double, c_int64, c_void_p]),
    "kvlc_corrected_attention_workspace": (c_size_t, [c_int64, c_int, c_int]),
    "kvlc_corrected_attention": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int,
                                         c_void_p, c_void_p, c_size_t, c_void_p]),
    "kvlc_decode_blocks": (c_int, [POINTER(KvlcCache), POINTER(KvlcAdapter), c_void_p, c_void_p, c_void_p,
                                   c_int32, POINTER(KvlcDecodeOpts), c_void_p, c_size_t, c_void_p]),
    "kvlc_ref_pack": (c_int, [c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p]),
    "kvlc_ref_unpack": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p]),
    "kvlc_ref_quantize": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_int, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "kvlc_ref_dequantize": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int, c_int,
                                    c_int, c_void_p, c_void_p]),
    "kvlc_ref_rotate": (c_int, [c_void_p, c_int64, c_int64, c_int, c_void_p, c_void_p]),
    "kvlc_ref_feature_map": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int, c_void_p,
                                     c_void_p]),
    "kvlc_ref_attention": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int,
                                   c_int, c_void_p, c_void_p, c_void_p]),
    "kvlc_ref_flush_scratch": (c_size_t, [c_int, c_int, c_int]),
    "kvlc_ref_flush": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p,
                               c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p]),
    "kvlc_ref_decode_scratch": (c_size_t, [c_int, c_int64, c_int64, c_int, c_int]),
    "kvlc_ref_decode": (c_int, [c_void_p, c_int, c_int, c_int, c_int, c_int64, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "kvlc_prefill_workspace": (c_size_t, [POINTER(KvlcCache), c_int64]),
    "kvlc_prefill": (c_int, [POINTER(KvlcCache), POINTER(KvlcAdapter), c_void_p, c_void_p, c_int64,
                             POINTER(c_int32), c_int32, c_void_p, c_size_t, c_void_p]),
    "kvlc_append_workspace": (c_size_t, [POINTER(KvlcCache)]),
    "kvlc_append": (c_int, [POINTER(KvlcCache), POINTER(KvlcAdapter), c_void_p, c_void_p,
                            POINTER(c_int32), POINTER(c_int32), c_void_p, c_size_t, c_void_p]),
    "kvlc_decode_workspace": (c_size_t, [POINTER(KvlcCache), POINTER(KvlcDecodeOpts)]),
    "kvlc_decode": (c_int, [POINTER(KvlcCache), POINTER(KvlcAdapter), c_void_p, c_void_p,
                            POINTER(KvlcDecodeOpts), c_void_p, c_size_t, c_void_p]),
    "kvlc_decode_partial": (c_int, [POINTER(KvlcCache), POINTER(KvlcAdapter), c_void_p, c_int32,
                                    c_int32, c_int32, c_void_p, c_void_p, POINTER(KvlcDecodeOpts),
                                    c_void_p, c_size_t, c_void_p]),
    "kvlc_stage_input": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "kvlc_merge_records": (c_int, [c_void_p, c_int32, c_int64, c_void_p, c_int32, c_int32, c_int32,
                                   c_int32, c_void_p, c_void_p]),
    "kvlc_export_chunk": (c_int, [POINTER(KvlcCache), c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "kvlc_unit_image_bytes": (c_size_t, [c_int32, c_int32, c_int32]),
    "kvlc_serialize_unit": (c_int, [POINTER(KvlcCache), c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p,
                                    c_void_p]),
    "kvlc_deserialize_unit": (c_int, [POINTER(KvlcCache), c_int32, c_void_p, c_int32, c_int32, c_int32,
                                      c_void_p]),
    "kvlc_quantize_pack": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_int, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p]),
    "kvlc_fwht_quantize_workspace": (c_size_t, [c_int64, c_int]),
    "kvlc_fwht_quantize_pack": (c_int, [c_void_p, c_int64, c_int, c_int64, c_int, c_int, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "kvlc_state_update_workspace": (c_size_t, [c_int64, c_int]),
    "kvlc_state_update": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "kvlc_flush_due": (c_int, [POINTER(KvlcCache), POINTER(KvlcAdapter), POINTER(c_int32), c_void_p,
                               c_size_t, c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    """Load libkvlinc.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make` or "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().kvlc_last_error().decode(errors="replace")


def call(name: str, *args):
    """Invoke a status-returning entry point; map codes to Python exceptions.

    KVLC_EINVAL carries the reference's ValueError text and raises ValueError,
    like the reference API does.
    """
    rc = getattr(load(), name)(*args)
    if rc == KVLC_OK:
        return
    msg = last_error()
    if rc == KVLC_EINVAL:
        raise ValueError(msg)
    raise KvlcError(f"{name}: {msg} (code {rc})")


def device_ok() -> bool:
    return bool(load().kvlc_device_ok())


def require_device():
    """Fail loudly: the product path has no CPU implementation."""
    import torch
    if not torch.cuda.is_available() or not device_ok():
        raise KvlcError("libkvlinc needs an sm_100 (B200) CUDA device; there is no CPU fallback")


def ptr(t) -> int:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream
