"""GraphSAGE-style minibatch sampling with CUDA graphs (nd_khop_plan_*).

Training loops sample many equal-size batches: k-hop (fanouts) over a
batch of roots (driver.py:203-235 per batch; SURVEY §8(d) C3's 1,024-root
batches).  A ``KhopBatchSampler`` captures the fixed-layout k-hop run for
one batch size into a CUDA graph over preallocated buffers; each
``sample()`` is then one device parameter write, one roots copy and one
graph launch on the current stream (no allocation, no host
synchronisation).  The rows equal ``run_device`` of the same batch (same
roots, same sample ids: the keyed RNG).

    sampler = KhopBatchSampler(graph, fanouts=[25, 10], batch_size=1024)
    off, ids, blocks = sampler.sample(roots, sample_lo=b * 1024, seed=7)
    # off: int64 [n+1] device; ids[:off[-1]]: roots then sampled vertices;
    # blocks[k]: int32 [n, B_k] step-k slots (-1 = NULL), the dense layout
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from .graph import as_device_graph


class KhopBatchSampler:
    def __init__(self, graph, fanouts, batch_size: int, stream=None):
        import numpy as np
        torch = _lib.require_cuda()
        L = _lib.load()
        self.dg = as_device_graph(graph)
        self.fanouts = [int(f) for f in fanouts]
        self.n = int(batch_size)
        fan = np.ascontiguousarray(self.fanouts, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(L.nd_khop_plan_create(self.dg.handle, _lib.ptr(fan), len(fan), self.n,
                                         _lib.stream_ptr(stream), C.byref(h)), "nd_khop_plan_create")
        self._h = h
        S = len(self.fanouts)
        roots, off, ids = C.c_void_p(), C.c_void_p(), C.c_void_p()
        cap = C.c_int64()
        blocks = (C.c_void_p * S)()
        sizes = (C.c_int64 * S)()
        _lib.check(L.nd_khop_plan_outputs(h, C.byref(roots), C.byref(off), C.byref(ids), C.byref(cap),
                                          blocks, sizes, S))
        from .graph import device_view
        self.cap = cap.value
        self.roots = device_view(roots.value, self.n, "int64", self)
        self.final_off = device_view(off.value, self.n + 1, "int64", self)
        self.final_ids = device_view(ids.value, self.cap, "int32", self)
        widths, b = [], 1
        for f in self.fanouts:
            b *= f
            widths.append(b)
        self.blocks = [device_view(blocks[k], sizes[k], "int32", self).view(self.n, widths[k])
                       for k in range(S)]
        self._torch = torch

    def sample(self, roots=None, sample_lo: int = 0, seed: int = 0, stream=None):
        """One batch: `roots` a device int64 tensor [batch_size] (None: the
        sampler's own `roots` buffer, already filled).  Returns (final_off,
        final_ids, blocks) device views, valid until the next sample()."""
        if roots is not None:
            if roots.dtype != self._torch.int64 or roots.numel() != self.n or not roots.is_cuda:
                raise ValueError(f"roots must be a CUDA int64 tensor of {self.n} vertices")
            roots = roots.contiguous()
        _lib.check(_lib.load().nd_khop_plan_run(self._h, _lib.ptr(roots), int(sample_lo),
                                                C.c_uint64(int(seed) & (2**64 - 1)),
                                                _lib.stream_ptr(stream)), "nd_khop_plan_run")
        return self.final_off, self.final_ids, self.blocks

    def close(self):
        if self._h is not None and _lib._lib is not None:
            _lib._lib.nd_khop_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
