"""Row sharding of CER/CSER encodings over the GPUs of one node.

Rows of a CER/CSER matrix are independent: a shard is a contiguous row
block ``[r0, r1)`` cut out of the global encoding (not a re-encode) —

* ``row_ptr[r0..r1]`` rebased by ``row_ptr[r0]``,
* ``omega_ptr[row_ptr[r0]..row_ptr[r1]]`` rebased by its first entry,
* the matching ``col_index`` span (and CSER ``omega_index`` span),
* ``omega`` unchanged (CER ranks are row-relative, CSER indices global).

The activations are replicated, each rank computes its block of y, and the
only exchange is one all-gather of the y blocks.  Two exchanges:

* ``RowShardedDot``: the local dot, then ``all_gather_into_tensor`` (NCCL over
  NVLink on a GPU node; gloo in the CPU tests), optionally left in flight
  (``start``/``wait``) so the next product's kernel overlaps it;
* ``PeerRowShardedDot``: the all-gather fused into the dot kernels' epilogue
  (``cerdot_dot_peers``): every finished y element is stored straight into
  every rank's output buffer over NVLink peer mappings of a torch
  symmetric-memory buffer, then one stream-ordered signal/wait barrier.

Block boundaries come from ``cerdot_shard_plan`` (balanced encoded bytes).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .formats import CerMatrix, CserMatrix


def plan_rows(enc, parts: int) -> list[int]:
    """parts+1 row bounds balancing encoded bytes (cerdot_shard_plan)."""
    rp = np.ascontiguousarray(enc.row_ptr)
    op = np.ascontiguousarray(enc.omega_ptr)
    bounds = (ctypes.c_int64 * (parts + 1))()
    oi_bits = enc.omega_index_bits if isinstance(enc, CserMatrix) else 0
    _native.check(_native.lib().cerdot_shard_plan(rp.ctypes.data, rp.dtype.itemsize * 8, op.ctypes.data,
                                                  op.dtype.itemsize * 8, enc.col_index_bits, oi_bits, enc.m,
                                                  parts, bounds))
    return list(bounds)


def even_rows(m: int, parts: int) -> list[int]:
    return [m * p // parts for p in range(parts + 1)]


def slice_rows(enc, r0: int, r1: int):
    """Rows [r0, r1) of an encoding as a self-contained encoding (host arrays; uploads on first dot)."""
    if not 0 <= r0 <= r1 <= enc.m:
        raise ValueError(f"row block [{r0}, {r1}) out of range for m={enc.m}")
    rp = enc.row_ptr.astype(np.int64)
    op = enc.omega_ptr.astype(np.int64)
    s0, s1 = int(rp[r0]), int(rp[r1])
    e0, e1 = int(op[s0]), int(op[s1])
    row_ptr = (rp[r0:r1 + 1] - s0).astype(enc.row_ptr.dtype)
    omega_ptr = (op[s0:s1 + 1] - e0).astype(enc.omega_ptr.dtype)
    col = enc.col_index[e0:e1]
    if isinstance(enc, CserMatrix):
        return CserMatrix(enc.omega, col, enc.omega_index[s0:s1], omega_ptr, row_ptr, r1 - r0, enc.n,
                          enc.element_bits, enc.mode_index)
    return CerMatrix(enc.omega, col, omega_ptr, row_ptr, r1 - r0, enc.n, enc.element_bits)


def slice_rows_device(enc, r0: int, r1: int):
    """Rows [r0, r1) of a DEVICE-resident encoding as a new device-resident encoding, cut on the device
    (no host round trip of the index arrays): the same slice as ``slice_rows`` -- rowPtr / omegaPtr
    rebased, the colI (and CSER omegaI) spans copied, omega unchanged, the global widths kept -- plus the
    derived rowEntry index of the block."""
    import torch

    from .device import DeviceEncoding, torch_mod  # noqa: F401

    dev = enc.device_encoding()
    if not 0 <= r0 <= r1 <= dev.m:
        raise ValueError(f"row block [{r0}, {r1}) out of range for m={dev.m}")
    tdt = {8: torch.uint8, 16: torch.uint16, 32: torch.uint32}

    def view(name, start, stop):
        b = dev.bits[name] // 8
        o = dev.offsets[name]
        return dev.arena[o + start * b: o + stop * b].view(tdt[dev.bits[name]])

    rp = view("rowPtr", r0, r1 + 1).to(torch.int64)
    s0, s1 = int(rp[0]), int(rp[-1])
    op = view("omegaPtr", s0, s1 + 1).to(torch.int64)
    e0, e1 = int(op[0]), int(op[-1])
    m, segs, nnz = r1 - r0, s1 - s0, e1 - e0
    offsets, total = DeviceEncoding.layout(dev.kind, m, dev.k, nnz, segs, dev.bits)
    arena = torch.zeros(total, dtype=torch.uint8, device=dev.device)

    def put(name, t):
        o = offsets[name]
        raw = t.contiguous().view(torch.uint8)
        arena[o: o + raw.numel()] = raw

    put("omega", dev.arena[dev.offsets["omega"]: dev.offsets["omega"] + 8 * dev.k])
    put("colI", view("colI", e0, e1))
    put("omegaPtr", (op - e0).to(tdt[dev.bits["omegaPtr"]]))
    put("rowPtr", (rp - s0).to(tdt[dev.bits["rowPtr"]]))
    if dev.kind == _native.CSER:
        put("omegaI", view("omegaI", s0, s1))
    seg_rows = rp[1:] - rp[:-1]
    nnz_rows = op[(rp[1:] - s0)] - op[(rp[:-1] - s0)] if m else seg_rows
    new = DeviceEncoding(dev.kind, m, dev.n, dev.k, nnz, segs, dev.mode_index, dev.background, dict(dev.bits), arena,
                         offsets, int(nnz_rows.max()) if m else 0, int(seg_rows.max()) if m else 0)
    with torch.cuda.device(dev.device):
        new.fill_row_entries(torch.cuda.current_stream(dev.device).cuda_stream)
    cls = type(enc)
    if isinstance(enc, CserMatrix):
        return cls(None, None, None, None, None, m, enc.n, enc.element_bits, enc.mode_index, _device=new)
    return cls(None, None, None, None, m, enc.n, enc.element_bits, _device=new)


class RowShardedDot:
    """y = A.x with A's rows split over the ranks of a process group.

    ``local`` is this rank's row block (an encoding, or any object accepted by
    ``compute``), ``rows_per_rank`` the block heights (all-gather needs equal
    blocks, so shorter blocks are padded).  ``compute(local, x)`` returns the
    local y block as a torch tensor on the communication device; it defaults
    to the CUDA dot (``kernels.dot_device``) and is injectable so the
    exchange logic can be exercised on CPU with gloo.
    """

    def __init__(self, local, rows_per_rank: list[int], group=None, compute=None):
        import torch.distributed as dist

        self.local = local
        self.rows = list(rows_per_rank)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if len(self.rows) != self.world:
            raise ValueError(f"{len(self.rows)} row blocks for a world of {self.world}")
        self.block = max(self.rows) if self.rows else 0
        if compute is None:
            from .kernels import dot_device

            compute = dot_device
        self.compute = compute
        self._gather = None

    def __call__(self, x):
        return self.start(x).wait()

    def start(self, x) -> "PendingRows":
        """Compute the local block and start the all-gather without waiting for it: work queued on the
        current stream afterwards (e.g. the next layer's local dot) overlaps the exchange.  ``wait()``
        on the result returns the full y (the current stream then waits for the collective)."""
        import torch
        import torch.distributed as dist

        y = self.compute(self.local, x)
        if self.world == 1:
            return PendingRows(y, None, None)
        shape = (self.block,) + tuple(y.shape[1:])
        if y.shape[0] != self.block:
            pad = torch.zeros(shape, dtype=y.dtype, device=y.device)
            pad[: y.shape[0]] = y
            y = pad
        out = torch.empty((self.world * self.block,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
        work = dist.all_gather_into_tensor(out, y.contiguous(), group=self.group, async_op=True)
        rows = None if all(r == self.block for r in self.rows) else (self.block, self.rows)
        return PendingRows(out, work, rows)


class PendingRows:
    """An in-flight row-sharded product (RowShardedDot.start)."""

    def __init__(self, out, work, rows):
        self._out, self._work, self._rows = out, work, rows

    def wait(self):
        import torch

        if self._work is not None:
            self._work.wait()
            self._work = None
        if self._rows is None:
            return self._out
        block, rows = self._rows
        return torch.cat([self._out[i * block: i * block + r] for i, r in enumerate(rows)], dim=0)


class PeerRowShardedDot:
    """y = A.x with A's rows split over the ranks, the y all-gather fused into the kernels (NVLink P2P).

    The output lives in a symmetric-memory buffer (``torch.distributed._symmetric_memory``) of
    world x block rows; the local dot writes its rows into its own block and, from the same epilogue
    stores, into the same rows of every peer's buffer (``cerdot_dot_peers``).  ``handle.barrier()``
    (stream-ordered signal/wait over the symmetric signal pads) then makes every rank's copy complete.
    The returned tensor is the symmetric buffer itself (rows of every rank), valid until the next call
    on ANY rank (peers write into it): consume or copy it before the ranks' next product, or rotate
    several instances (as bench.py does).
    """

    def __init__(self, local, rows_per_rank: list[int], batch: int = 1, group=None, device=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.local = local
        self.rows = list(rows_per_rank)
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        if len(self.rows) != self.world:
            raise ValueError(f"{len(self.rows)} row blocks for a world of {self.world}")
        self.block = max(self.rows)
        self.batch = int(batch)
        device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        shape = (self.world * self.block,) if self.batch == 1 else (self.world * self.block, self.batch)
        self.buf = symm_mem.empty(shape, dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self.buf, self.group)
        ptrs = [int(p) for i, p in enumerate(self.handle.buffer_ptrs) if i != self.rank]
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)
        r0 = self.rank * self.block
        self.y_local = self.buf[r0: r0 + self.rows[self.rank]]
        self.peer_offset = r0 * (1 if self.batch == 1 else self.batch)

    def __call__(self, x, barrier: bool = True):
        """``barrier=False`` leaves the exchange to a later call's barrier (one barrier after several
        products makes all of them complete: it orders every prior peer store of every rank)."""
        import torch

        from .kernels import dot_device

        dot_device(self.local, x, out=self.y_local, peers=self.peers, peer_offset=self.peer_offset)
        if barrier:
            self.handle.barrier(channel=0)
        if all(r == self.block for r in self.rows):
            return self.buf
        return torch.cat([self.buf[i * self.block: i * self.block + r] for i, r in enumerate(self.rows)], dim=0)
