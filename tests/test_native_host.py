"""CPU tests: the C-ABI library loads and exports its header, host logic, error mapping."""

import ctypes

import numpy as np
import pytest

import paper_1805_10692_b200 as cd
from conftest import has_gpu
from paper_1805_10692_b200 import _native, synth


def _golden(small_cases, name):
    return next(c for c in small_cases if c["name"] == name)


def _cer_from(g, m, n):
    return cd.CerMatrix(np.array(g["omega"]), np.array(g["colI"], dtype=np.uint8),
                        np.array(g["omegaPtr"], dtype=np.uint8), np.array(g["rowPtr"], dtype=np.uint8), m, n)


def _cser_from(g, m, n):
    return cd.CserMatrix(np.array(g["omega"]), np.array(g["colI"], dtype=np.uint8),
                         np.array(g["omegaI"], dtype=np.uint8), np.array(g["omegaPtr"], dtype=np.uint8),
                         np.array(g["rowPtr"], dtype=np.uint8), m, n, mode_index=g["mode_index"])


def test_library_exports_every_header_symbol():
    L = _native.lib()
    names = _native.header_functions()
    assert len(names) >= 11
    for name in names:
        assert hasattr(L, name), name
    assert L.cerdot_abi_version() == 3


def test_index_bitwidth_matches_reference_table():
    # tests/test_formats.py:121-127
    for value, bits in [(0, 8), (255, 8), (256, 16), (65535, 16), (65536, 32), (70000, 32)]:
        assert cd.index_bitwidth(value) == bits
    with pytest.raises(ValueError):
        cd.index_bitwidth(1 << 32)
    with pytest.raises(ValueError, match="unsigned"):
        cd.index_bitwidth(-1)


def test_shard_plan_balances_bytes():
    L = _native.lib()
    rng = np.random.default_rng(0)
    m = 1000
    segs = rng.integers(0, 20, size=m)
    row_ptr = np.concatenate(([0], np.cumsum(segs))).astype(np.uint32)
    sizes = rng.integers(0, 50, size=int(row_ptr[-1]))
    omega_ptr = np.concatenate(([0], np.cumsum(sizes))).astype(np.uint32)
    for oi_bits in (0, 8, 32):  # CER; CSER with u8 / u32 omegaI (counted per segment)
        for parts in (1, 2, 3, 8):
            b = (ctypes.c_int64 * (parts + 1))()
            assert L.cerdot_shard_plan(row_ptr.ctypes.data, 32, omega_ptr.ctypes.data, 32, 16, oi_bits, m, parts,
                                       b) == 0
            bounds = list(b)
            assert bounds[0] == 0 and bounds[-1] == m and all(x <= y for x, y in zip(bounds, bounds[1:]))
            per_row = np.array([2 * (omega_ptr[row_ptr[r + 1]] - omega_ptr[row_ptr[r]]) + (4 + oi_bits // 8) * segs[r]
                                + 4 for r in range(m)], dtype=float)
            shares = [per_row[a:c].sum() for a, c in zip(bounds[:-1], bounds[1:])]
            assert max(shares) - min(shares) <= 2 * per_row.max() + 1e-9
    b = (ctypes.c_int64 * 2)()
    assert L.cerdot_shard_plan(row_ptr.ctypes.data, 32, omega_ptr.ctypes.data, 32, 16, 0, m, 0, b) == _native.E_VALUE
    with pytest.raises(ValueError):
        _native.check(_native.E_VALUE)


def test_status_mapping():
    for status, exc in [(_native.E_VALUE, ValueError), (_native.E_TYPE, TypeError), (_native.E_INDEX, IndexError),
                        (_native.E_CUDA, RuntimeError), (_native.E_UNSUPPORTED, RuntimeError)]:
        with pytest.raises(exc):
            _native.check(status)
    _native.check(_native.OK)


def test_traces_from_host_arrays(small_cases):
    # tests/test_kernels.py:273-286: row-2 traces of M are 24 (CER) and 25 (CSER)
    case = _golden(small_cases, "M_ones")
    cer = _cer_from(case["cer"], 5, 12)
    cser = _cser_from(case["cser"], 5, 12)
    t = cd.row_trace(cer, 1)
    assert t.total() == 24
    assert t.by_kind() == {"read": 17, "mul": 1, "sum": 5, "write": 1}
    assert t.count("read", "rowPtr") == 2 and t.count("read", "omegaPtr") == 2
    assert t.count("read", "omega") == 1 and t.count("read", "colI") == 6 and t.count("read", "input") == 6
    t2 = cd.row_trace(cser, 1)
    assert t2.total() == 25 and t2.count("read", "omegaI") == 1
    t3 = cd.row_trace(cer, 0, input_bits=16, output_bits=32)
    assert t3.counts.get(("sum", 16, "none"), 0) == 4 and t3.counts.get(("sum", 32, "none"), 0) == 2
    full = cd.trace_of(cer)
    per_rows = cd.OpTrace()
    for r in range(5):
        per_rows = per_rows.merged(cd.row_trace(cer, r))
    for key in set(full.counts) | set(per_rows.counts):
        if key[0] != "other":
            assert full.counts.get(key, 0) == per_rows.counts.get(key, 0)
    t_cols = cd.trace_of(cer, columns=3)
    for key, cnt in full.counts.items():
        assert t_cols.counts[key] == 3 * cnt


def test_padding_trace(small_cases):
    # tests/test_kernels.py:304-312
    case = _golden(small_cases, "padding_rule")
    cer = _cer_from(case["cer"], 3, 3)
    t = cd.row_trace(cer, 1)
    assert t.count("read", "omegaPtr") == 3 and t.count("mul") == 1 and t.count("read", "omega") == 1


def test_storage_and_entry_counts(small_cases):
    case = _golden(small_cases, "M_ones")
    cer = _cer_from(case["cer"], 5, 12)
    cser = _cser_from(case["cser"], 5, 12)
    assert cd.entry_count(cer)["total"] == 49 and cd.entry_count(cser)["total"] == 59
    assert cd.entry_count(cd.DenseMatrix(np.zeros((5, 12))))["total"] == 60
    assert cd.storage_bits(cer) == case["cer"]["storage_bits"]
    assert cd.storage_bits(cser) == case["cser"]["storage_bits"]
    assert set(cd.array_bytes(cser)) == {"input", "output", "omega", "colI", "omegaI", "omegaPtr", "rowPtr"}


def test_encodings_are_immutable(small_cases):
    cer = _cer_from(_golden(small_cases, "M_ones")["cer"], 5, 12)
    with pytest.raises(AttributeError):
        cer.m = 3
    with pytest.raises(ValueError):
        cer.omega[0] = 1.0  # read-only view


def test_dense_containers():
    a = cd.DenseMatrix([[1, 2], [3, 4]])
    assert a.values.dtype == np.float64 and not a.values.flags.writeable and (a.m, a.n, a.size) == (2, 2, 4)
    with pytest.raises(ValueError):
        cd.DenseMatrix([1, 2])
    with pytest.raises(ValueError):
        cd.Vector([1.0], element_bits=12)


@pytest.mark.skipif(has_gpu(), reason="checks the no-CUDA behaviour")
def test_no_cpu_fallback():
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cd.encode_cer(np.eye(3))
    cer = cd.CerMatrix(np.array([0.0, 1.0]), np.array([0], np.uint8), np.array([0, 1], np.uint8),
                       np.array([0, 1], np.uint8), 1, 1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        cd.dot_cer(cer, np.ones(1))
    with pytest.raises(ValueError, match="mismatch"):  # argument errors come first, like the reference
        cd.dot_cer(cer, np.ones(3))


def test_synth_chunked_generation_equals_single_draw():
    cfg = synth.config("oracle")
    rng = np.random.default_rng(0)
    one = synth.levels_of(cfg)[rng.choice(cfg.k, size=(cfg.m, cfg.n), p=synth.pmf_of(cfg))]
    chunked = synth.make_weights(cfg, np.random.default_rng(0), chunk_rows=37)
    assert np.array_equal(one, chunked)
    assert synth.levels_of(cfg)[cfg.k // 2] == 0.0


def test_synth_config_sizes_match_survey():
    # config 1 nnz 78,678, CER segments 6,910, CSER 6,264
    from oracle import c_oracle

    w, _ = synth.make_layer("oracle")
    cer = c_oracle.encode(w, "cer")
    cser = c_oracle.encode(w, "cser")
    assert cer["colI"].size == 78678
    assert cer["omegaPtr"].size - 1 == 6910 and cser["omegaPtr"].size - 1 == 6264
