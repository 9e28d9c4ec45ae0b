"""Sample-set output and its text layouts (mirror of trawl/output.py:27-150).

A run's output stays compact: roots plus either per-sample *chains*
(walk apps: one slot per step, engine/chain.py:167-179) or per-step slot
blocks (multi-slot and collective apps, driver.py:93-131), plus recorded
edges.  The device engine fills these arrays (and the compacted
final-layout rows ``final_off``/``final_ids``) in HBM; the host view here
copies them once and derives the reference's ``final_rows`` /
``step_rows`` / ``render_text`` views on demand.
"""

from __future__ import annotations

import struct
from typing import Optional

import numpy as np

from .core import NULL_VERTEX, Sample

LAYOUT_FINAL = "final"
LAYOUT_PER_STEP = "per-step"
OUTPUT_MAGIC = b"NDSO"
OUTPUT_VERSION = 1

_E = np.empty(0, dtype=np.int64)


def _offsets(counts) -> np.ndarray:
    off = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off


class SampleSetOutput:
    """Results of one engine run (output.py:43-69 semantics).

    Storage (host numpy, int64):
      sample_ids[N]; roots_off[N+1], roots (final root sets)
      chain mode:  chain_off[N+1], chain_vals (NULLs kept)
      steps mode:  step_counts[S, N] slots per sample, step_vals step-major
      rec_counts[S, N], rec_t, rec_v (recorded edges, step-major) or None
      final_off/final_ids: compacted final rows (dense ids) when the device
      produced them, else derived.
    """

    def __init__(self, sample_ids, roots_off, roots, n_steps, remap=None, stats=None, *,
                 chain_off=None, chain_vals=None, step_counts=None, step_vals=None,
                 rec_counts=None, rec_t=None, rec_v=None, final_off=None, final_ids=None):
        self.sample_ids = np.asarray(sample_ids, dtype=np.int64)
        self.roots_off = np.asarray(roots_off, dtype=np.int64)
        self.roots = np.asarray(roots, dtype=np.int64)
        self.n_steps = int(n_steps)
        self.remap = remap
        self.stats = stats
        self.chain_off = None if chain_off is None else np.asarray(chain_off, dtype=np.int64)
        self.chain_vals = None if chain_vals is None else np.asarray(chain_vals, dtype=np.int64)
        self.step_counts = None if step_counts is None else np.asarray(step_counts, dtype=np.int64)
        self.step_vals = None if step_vals is None else np.asarray(step_vals, dtype=np.int64)
        self.rec_counts = rec_counts
        self.rec_t = rec_t
        self.rec_v = rec_v
        self._final = None
        if final_off is not None:
            self._final = (np.asarray(final_off, dtype=np.int64), np.asarray(final_ids, dtype=np.int64))
        self._samples = None

    # -- sizes --------------------------------------------------------------
    @property
    def n_samples(self) -> int:
        return len(self.sample_ids)

    def _step_base(self) -> np.ndarray:
        """[S+1] start of each step block in step_vals."""
        return _offsets(self.step_counts.sum(axis=1)) if self.step_counts is not None else _E

    def total_sampled(self) -> int:
        if self.chain_vals is not None:
            return int((self.chain_vals != NULL_VERTEX).sum())
        if self.step_vals is not None:
            return int((self.step_vals != NULL_VERTEX).sum())
        return 0

    def total_recorded(self) -> int:
        return 0 if self.rec_t is None else len(self.rec_t)

    # -- final layout ---------------------------------------------------------
    def final_csr(self):
        """(offsets[N+1], ids) of roots followed by every non-NULL sampled
        vertex in step order — dense ids (core.py:116-123)."""
        if self._final is None:
            self._final = self._derive_final()
        return self._final

    def _derive_final(self):
        N = self.n_samples
        rlen = np.diff(self.roots_off)
        if self.chain_vals is not None:
            clen = np.diff(self.chain_off)
            owner = np.repeat(np.arange(N), clen)
            keep = self.chain_vals != NULL_VERTEX
            nn = np.bincount(owner[keep], minlength=N)
            off = _offsets(rlen + nn)
            ids = np.empty(off[-1], dtype=np.int64)
            # roots
            rpos = off[:-1].repeat(rlen) + (np.arange(len(self.roots)) - self.roots_off[:-1].repeat(rlen))
            ids[rpos] = self.roots
            kv = self.chain_vals[keep]
            ko = owner[keep]
            rank = np.arange(len(kv)) - _offsets(nn)[:-1][ko]
            ids[off[:-1][ko] + rlen[ko] + rank] = kv
            return off, ids
        parts_len = rlen.copy()
        if self.step_vals is not None and len(self.step_vals):
            S = self.step_counts.shape[0]
            owner = np.concatenate([np.repeat(np.arange(N), self.step_counts[s]) for s in range(S)])
            keep = self.step_vals != NULL_VERTEX
            nn = np.bincount(owner[keep], minlength=N)
            parts_len = parts_len + nn
            off = _offsets(parts_len)
            ids = np.empty(off[-1], dtype=np.int64)
            rpos = off[:-1].repeat(rlen) + (np.arange(len(self.roots)) - self.roots_off[:-1].repeat(rlen))
            ids[rpos] = self.roots
            kv = self.step_vals[keep]
            ko = owner[keep]
            # stable order per sample: step-major storage is already step order
            order = np.argsort(ko, kind="stable")
            kv, ko = kv[order], ko[order]
            rank = np.arange(len(kv)) - _offsets(nn)[:-1][ko]
            ids[off[:-1][ko] + rlen[ko] + rank] = kv
            return off, ids
        return self.roots_off.copy(), self.roots.copy()

    def final_rows(self) -> list[np.ndarray]:
        off, ids = self.final_csr()
        ids = self._remap(ids)
        return [ids[off[i]:off[i + 1]] for i in range(self.n_samples)]

    def _remap(self, ids):
        if self.remap is None:
            return ids
        return np.asarray(self.remap)[ids]

    # -- per-step layout --------------------------------------------------------
    def step_csr(self, step: int):
        """(offsets[N+1], ids) of one step's non-NULL vertices (-1 = roots)."""
        N = self.n_samples
        if step == -1:
            return self.roots_off, self.roots
        if self.chain_vals is not None:
            clen = np.diff(self.chain_off)
            has = clen > step
            v = np.full(N, NULL_VERTEX, dtype=np.int64)
            v[has] = self.chain_vals[self.chain_off[:-1][has] + step]
            keep = v != NULL_VERTEX
            return _offsets(keep.astype(np.int64)), v[keep]
        if self.step_counts is None or step >= self.step_counts.shape[0]:
            return np.zeros(N + 1, dtype=np.int64), _E
        base = self._step_base()[step]
        cnt = self.step_counts[step]
        block = self.step_vals[base:base + cnt.sum()]
        owner = np.repeat(np.arange(N), cnt)
        keep = block != NULL_VERTEX
        return _offsets(np.bincount(owner[keep], minlength=N)), block[keep]

    def step_rows(self, step: int) -> list[np.ndarray]:
        off, ids = self.step_csr(step)
        ids = self._remap(ids)
        return [ids[off[i]:off[i + 1]] for i in range(self.n_samples)]

    def total_vertices(self) -> int:
        off, _ = self.final_csr()
        return int(off[-1])

    # -- reference object view -------------------------------------------------
    @property
    def samples(self) -> list[Sample]:
        """Per-sample ``Sample`` objects (step slot arrays with NULLs, recorded
        edges) — built lazily for API compatibility."""
        if self._samples is None:
            self._samples = self._build_samples()
        return self._samples

    def _build_samples(self):
        N = self.n_samples
        out = []
        if self.step_counts is not None:
            sb = self._step_base()
            soff = [sb[s] + _offsets(self.step_counts[s]) for s in range(self.step_counts.shape[0])]
        if self.rec_counts is not None and self.rec_t is not None:
            rb = _offsets(np.asarray(self.rec_counts).sum(axis=1))
            roff = [rb[s] + _offsets(self.rec_counts[s]) for s in range(len(self.rec_counts))]
        for i in range(N):
            s = Sample(self.sample_ids[i], self.roots[self.roots_off[i]:self.roots_off[i + 1]])
            if self.chain_vals is not None:
                ch = self.chain_vals[self.chain_off[i]:self.chain_off[i + 1]]
                s.step_vertices = [ch[k:k + 1] for k in range(len(ch))]
            elif self.step_counts is not None:
                for st in range(self.step_counts.shape[0]):
                    c = self.step_counts[st, i]
                    if c == 0 and not any(self.step_counts[st2, i] for st2 in range(st, self.step_counts.shape[0])):
                        break
                    s.step_vertices.append(self.step_vals[soff[st][i]:soff[st][i + 1]])
            if self.rec_counts is not None and self.rec_t is not None:
                for st in range(len(self.rec_counts)):
                    a, b = roff[st][i], roff[st][i + 1]
                    s.recorded_edges.append((self.rec_t[a:b], self.rec_v[a:b]))
            out.append(s)
        return out


# ---------------------------------------------------------------------------
# text / binary writers (output.py:72-150)

def _fmt_rows(sample_ids, off, ids, lines):
    for i, sid in enumerate(sample_ids):
        row = ids[off[i]:off[i + 1]]
        lines.append(f"{int(sid)}: " + " ".join(map(str, row.tolist())))


# outputs with at least this many ids are printed on the GPU (nd_format_rows)
DEVICE_FORMAT_MIN_IDS = 1 << 16


def _device_rows_text(sample_ids, off, ids, remap):
    """The block's text lines printed on the device (nd_format_rows, one
    warp per row), byte-identical to _fmt_rows, as a uint8 array (any
    bytes-like use: file writes, b"".join, bytes()); None without CUDA."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    if not torch.cuda.is_available():
        return None
    import ctypes as C

    from . import _lib
    L = _lib.load()
    ids = np.asarray(ids)
    ids = ids if ids.dtype in (np.int32, np.int64) else ids.astype(np.int64)
    d_off = torch.from_numpy(np.ascontiguousarray(off, dtype=np.int64)).cuda()
    d_ids = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
    d_sid = torch.from_numpy(np.ascontiguousarray(sample_ids, dtype=np.int64)).cuda()
    d_map = None if remap is None else torch.from_numpy(
        np.ascontiguousarray(remap, dtype=np.int64)).cuda()
    n = len(off) - 1
    tl = C.c_int64()
    args = (_lib.ptr(d_off), _lib.ptr(d_ids), ids.dtype.itemsize, _lib.ptr(d_sid), n,
            _lib.ptr(d_map), _lib.stream_ptr())
    _lib.check(L.nd_format_rows(*args, None, 0, C.byref(tl)), "nd_format_rows")
    # a pageable buffer: pinning a GB-sized one costs more than the slower copy
    buf = np.empty(tl.value, dtype=np.uint8)
    _lib.check(L.nd_format_rows(*args, _lib.ptr(buf), tl.value, C.byref(tl)), "nd_format_rows")
    return buf


def _rows_bytes(output: "SampleSetOutput", off, ids):
    """One block's lines (each ending in a newline), bytes-like."""
    if len(ids) >= DEVICE_FORMAT_MIN_IDS:
        text = _device_rows_text(output.sample_ids, off, ids, output.remap)
        if text is not None:
            return text
    lines = []
    _fmt_rows(output.sample_ids, off, output._remap(ids), lines)
    return "".join(line + "\n" for line in lines).encode()


def _render_parts(output: SampleSetOutput, layout: str) -> list:
    parts = [f"# layout={layout}\n".encode()]
    if layout == LAYOUT_FINAL:
        off, ids = output.final_csr()
        parts.append(_rows_bytes(output, off, ids))
    elif layout == LAYOUT_PER_STEP:
        if output.n_samples:
            parts.append(b"roots:\n")
            off, ids = output.step_csr(-1)
            parts.append(_rows_bytes(output, off, ids))
            for st in range(output.n_steps):
                parts.append(f"step {st}:\n".encode())
                off, ids = output.step_csr(st)
                parts.append(_rows_bytes(output, off, ids))
    else:
        raise ValueError(f"unknown layout {layout!r}")
    return parts


def render_bytes(output: SampleSetOutput, layout: str) -> bytes:
    """render_text as UTF-8 bytes; large blocks are printed on the GPU."""
    return b"".join(_render_parts(output, layout))


def render_text(output: SampleSetOutput, layout: str) -> str:
    """The reference's text layouts (output.py:72-92)."""
    return render_bytes(output, layout).decode()


def emit(output: SampleSetOutput, layout: str, path) -> None:
    with open(path, "wb") as fh:
        for part in _render_parts(output, layout):
            fh.write(part)


def write_binary(output: SampleSetOutput, layout: str, path) -> None:
    """NDSO layout (output.py:108-124)."""
    if layout == LAYOUT_FINAL:
        blocks = [output.final_csr()]
    else:
        blocks = [output.step_csr(s) for s in range(-1, output.n_steps)]
    with open(path, "wb") as fh:
        fh.write(OUTPUT_MAGIC)
        fh.write(struct.pack("<II", OUTPUT_VERSION, 0 if layout == LAYOUT_FINAL else 1))
        fh.write(struct.pack("<QQ", output.n_samples, len(blocks)))
        for off, ids in blocks:
            fh.write(np.asarray(off, dtype="<u8").tobytes())
            fh.write(np.asarray(output._remap(ids), dtype="<i8").tobytes())


def write_remap(remap: np.ndarray, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("# dense original\n")
        for dense, orig in enumerate(remap):
            fh.write(f"{dense} {int(orig)}\n")


def dedup_rows(vals: np.ndarray) -> np.ndarray:
    """Sorted distinct non-NULL values (output.py:27-31)."""
    return np.unique(vals[vals != NULL_VERTEX])


def fallback_check(n_distinct: int, m_i: int) -> bool:
    """SP-fallback hint after a unique step (output.py:34-40)."""
    return 0 < n_distinct < m_i
