"""Row sharding + output all-gather, exercised with world_size 2 on CPU (gloo).

The device kernels are replaced by the pinned C oracle through RowShardedDot's
``compute`` hook, so this covers the planner (cerdot_shard_plan), the
encoding slicer and the exchange logic exactly as the NCCL path runs them.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1805_10692_b200 as cd
from oracle import c_oracle, numpy_port
from paper_1805_10692_b200 import shard, synth


def _as_dict(enc):
    out = {"kind": "cer" if isinstance(enc, cd.CerMatrix) else "cser", "m": enc.m, "n": enc.n,
           "omega": enc.omega, "colI": enc.col_index, "omegaPtr": enc.omega_ptr, "rowPtr": enc.row_ptr}
    if out["kind"] == "cser":
        out["omegaI"] = enc.omega_index
        out["mode_index"] = enc.mode_index
    return out


def _host_encoding(kind, w):
    e = numpy_port.encode_cer(w) if kind == "cer" else numpy_port.encode_cser(w)
    if kind == "cer":
        return cd.CerMatrix(e["omega"], e["colI"], e["omegaPtr"], e["rowPtr"], e["m"], e["n"])
    return cd.CserMatrix(e["omega"], e["colI"], e["omegaI"], e["omegaPtr"], e["rowPtr"], e["m"], e["n"],
                         mode_index=e["mode_index"])


def _oracle_compute(enc, x):
    return torch.from_numpy(c_oracle.dot(_as_dict(enc), x.numpy()))


def _worker(rank, world, port, kind, balanced, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, xs = synth.make_layer("oracle")
        full = _host_encoding(kind, w)
        bounds = shard.plan_rows(full, world) if balanced else shard.even_rows(full.m, world)
        local = shard.slice_rows(full, bounds[rank], bounds[rank + 1])
        rows = [bounds[i + 1] - bounds[i] for i in range(world)]
        op = shard.RowShardedDot(local, rows, compute=_oracle_compute)
        x = torch.from_numpy(np.stack([xs[1], -xs[1], 2 * xs[1]], axis=1).astype(np.float64))
        y = op(x)
        if rank == 0:
            np.save(result_path, y.numpy())
    finally:
        dist.destroy_process_group()


def _worker_overlap(rank, world, port, result_path):
    """CER and CSER products started back to back (two all-gathers in flight), then waited."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, xs = synth.make_layer("oracle")
        ops = []
        for kind in ("cer", "cser"):
            full = _host_encoding(kind, w)
            bounds = shard.plan_rows(full, world)
            local = shard.slice_rows(full, bounds[rank], bounds[rank + 1])
            ops.append(shard.RowShardedDot(local, [bounds[i + 1] - bounds[i] for i in range(world)],
                                           compute=_oracle_compute))
        x = torch.from_numpy(xs[1].astype(np.float64))
        pending = [op.start(x) for op in ops]
        ys = [p.wait() for p in pending]
        if rank == 0:
            np.save(result_path, np.stack([y.numpy() for y in ys]))
    finally:
        dist.destroy_process_group()


def test_overlapped_products_world2(tmp_path):
    out = str(tmp_path / "y2.npy")
    mp.spawn(_worker_overlap, args=(2, _free_port(), out), nprocs=2, join=True)
    w, xs = synth.make_layer("oracle")
    got = np.load(out)
    for i, kind in enumerate(("cer", "cser")):
        assert np.array_equal(got[i], c_oracle.dot(_as_dict(_host_encoding(kind, w)), xs[1].astype(np.float64)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind,balanced", [("cer", True), ("cser", True), ("cer", False)])
def test_row_sharded_dot_world2(tmp_path, kind, balanced):
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(2, _free_port(), kind, balanced, out), nprocs=2, join=True)
    w, xs = synth.make_layer("oracle")
    x = np.stack([xs[1], -xs[1], 2 * xs[1]], axis=1).astype(np.float64)
    ref = c_oracle.dot(_as_dict(_host_encoding(kind, w)), x)
    # rows are independent and the loop oracle is per-row: sharded == unsharded bitwise
    assert np.array_equal(np.load(out), ref)


def test_row_sharded_dot_world3_uneven(tmp_path):
    """Three ranks, byte-balanced blocks of unequal heights (all-gather of padded blocks), CSER."""
    out = str(tmp_path / "y3.npy")
    mp.spawn(_worker, args=(3, _free_port(), "cser", True, out), nprocs=3, join=True)
    w, xs = synth.make_layer("oracle")
    x = np.stack([xs[1], -xs[1], 2 * xs[1]], axis=1).astype(np.float64)
    ref = c_oracle.dot(_as_dict(_host_encoding("cser", w)), x)
    assert np.array_equal(np.load(out), ref)


def test_slices_are_valid_encodings():
    w, xs = synth.make_layer("oracle")
    for kind in ("cer", "cser"):
        full = _host_encoding(kind, w)
        for parts in (1, 3, 7):
            bounds = shard.plan_rows(full, parts)
            assert bounds[0] == 0 and bounds[-1] == full.m
            pieces = [shard.slice_rows(full, a, b) for a, b in zip(bounds[:-1], bounds[1:])]
            assert sum(p.nnz for p in pieces) == full.nnz
            assert sum(p.segment_count for p in pieces) == full.segment_count
            for p in pieces:
                assert int(p.row_ptr[0]) == 0 and int(p.omega_ptr[0]) == 0
                assert int(p.omega_ptr[-1]) == p.nnz and int(p.row_ptr[-1]) == p.segment_count
            ys = [c_oracle.dot(_as_dict(p), xs[1]) for p in pieces]
            assert np.array_equal(np.concatenate(ys), c_oracle.dot(_as_dict(full), xs[1]))
    with pytest.raises(ValueError):
        shard.slice_rows(full, 5, 2)


def test_uneven_blocks_are_padded_for_all_gather():
    # RowShardedDot pads short blocks to the longest; world of 1 short-circuits
    op = shard.RowShardedDot(object(), [4], compute=lambda enc, x: torch.arange(4.0))
    assert op(torch.zeros(3)).tolist() == [0.0, 1.0, 2.0, 3.0]


@pytest.mark.parametrize("kind", ["cer", "cser"])
def test_row_sharded_dot_world4_global_encoding(tmp_path, kind):
    """bench.py's N>1 layout at world 4: one GLOBAL encoding (one alphabet), byte-balanced row slices of it
    (the planner counts CSER omegaI bytes), y assembled by the all-gather: sharded == unsharded bitwise."""
    out = str(tmp_path / "y4.npy")
    mp.spawn(_worker, args=(4, _free_port(), kind, True, out), nprocs=4, join=True)
    w, xs = synth.make_layer("oracle")
    x = np.stack([xs[1], -xs[1], 2 * xs[1]], axis=1).astype(np.float64)
    ref = c_oracle.dot(_as_dict(_host_encoding(kind, w)), x)
    assert np.array_equal(np.load(out), ref)
