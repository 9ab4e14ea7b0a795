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


class AttnProxy:
    """Paged decode attention over a fixed set of live requests (bench interference
    workload proxy, NEXT-4): tables = [(pool_tensor_index, len, block_ids)], pools = the
    stage pools (torch int16 tensors).  run(stream) launches one kernel."""

    def __init__(self, pools, tables, L, H, B, d, qpk=4, device=None):
        import torch
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        ptrs = np.array([p.data_ptr() for p in pools], dtype=np.uint64)
        self.pools = torch.as_tensor(ptrs.view(np.int64)).to(self.dev)
        self.keep = pools
        rp, rl, ro, bts = [], [], [], []
        for pi, ln, blocks in tables:
            rp.append(pi)
            rl.append(ln)
            ro.append(len(bts))
            bts.extend(blocks)
        i32 = lambda x: torch.as_tensor(np.asarray(x, dtype=np.int32)).to(self.dev)
        self.rp, self.rl, self.ro, self.bt = i32(rp), i32(rl), i32(ro), i32(bts or [0])
        self.n, self.L, self.H, self.B, self.d, self.qpk = len(rp), L, H, B, d, qpk
        g = torch.Generator(device=self.dev).manual_seed(7)
        self.q = torch.randn(max(1, self.n * L * H * qpk * d), device=self.dev, generator=g)
        self.out = torch.empty_like(self.q)
        self.tokens = sum(rl)
        L_ = lib()
        L_.kvgen_attn_proxy.restype = ctypes.c_int
        L_.kvgen_attn_proxy.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int] * 6 + \
            [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]

    def run(self, stream: int) -> None:
        if self.n == 0:
            return
        rc = lib().kvgen_attn_proxy(self.pools.data_ptr(), self.rp.data_ptr(), self.rl.data_ptr(),
                                    self.ro.data_ptr(), self.bt.data_ptr(), self.n, self.L,
                                    self.H, self.B, self.d, self.qpk, self.q.data_ptr(),
                                    self.out.data_ptr(), stream)
        if rc != 0:
            raise RuntimeError("kvgen_attn_proxy failed")
