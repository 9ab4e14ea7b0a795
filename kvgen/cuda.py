"""CUDA twin of ``kvgen.content`` (device-side synthetic KV, for large configs).

Loads ``kvgen/libkvgen.so`` (built by ``__graft_entry__.build()``).  Input
generation only: the bench and the GPU tests use it to produce the dense
new-token KV that ``kv_append`` consumes, without a host round trip.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libkvgen.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run __graft_entry__.build()")
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.kvgen_content.restype = ctypes.c_int
        _lib.kvgen_content.argtypes = [ctypes.c_ulonglong, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return _lib


def content_tokens_cuda(seed: int, req_ids, positions, layer0: int, layers: int, kv_heads: int,
                        head_dim: int, out=None, stream=None, device=None):
    """Dense uint16-as-int16 torch tensor [n][L][2][H][d] on the device (same words as numpy)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    req = torch.as_tensor(np.asarray(req_ids, dtype=np.int64)).to(dev, non_blocking=False)
    pos = torch.as_tensor(np.asarray(positions, dtype=np.int32)).to(dev, non_blocking=False)
    n = int(req.numel())
    if out is None:
        out = torch.empty((n, layers, 2, kv_heads, head_dim), dtype=torch.int16, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
    rc = lib().kvgen_content(seed & ((1 << 64) - 1), req.data_ptr(), pos.data_ptr(), n, layer0,
                             layers, kv_heads, head_dim, out.data_ptr(), s)
    if rc != 0:
        raise RuntimeError(f"kvgen_content failed ({rc})")
    out._kvgen_keepalive = (req, pos)  # inputs must outlive the async kernel
    return out


def r9_observe(meta_ptr: int, replica_ptr: int, R: int, M: int, B: int, block_bytes: int,
               seg_bytes: int, n_obs: int, last_seq: int, max_spin: int = 1 << 28, device=None,
               stream=None):
    """Launch the concurrent R9 reader (test support, see kvgen.cu); returns
    (records tensor [n_obs][rec_bytes] uint8, n_done tensor, rec_bytes) -- read after sync."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    rec = 16 + 12 * R + R * seg_bytes
    rec = (rec + 15) // 16 * 16
    out = torch.zeros((n_obs, rec), dtype=torch.uint8, device=dev)
    n_done = torch.zeros(1, dtype=torch.int32, device=dev)
    L = lib()
    L.kvgen_r9_observe.restype = ctypes.c_int
    L.kvgen_r9_observe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_void_p,
                                   ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p]
    s = torch.cuda.current_stream(dev).cuda_stream if stream is None else stream
    rc = L.kvgen_r9_observe(meta_ptr, replica_ptr, R, M, B, block_bytes, seg_bytes, n_obs,
                            max_spin, last_seq, out.data_ptr(), rec, n_done.data_ptr(), s)
    if rc != 0:
        raise RuntimeError("kvgen_r9_observe failed")
    return out, n_done, rec
