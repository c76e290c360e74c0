"""The seeded synthetic layers: reproducible, chunk-independent, and the sizes the
survey probed (nnz and segment counts of the configs)."""

import numpy as np
import pytest

from oracle import numpy_port
from paper_1805_10692_b200 import synth


def test_chunked_draw_equals_one_call():
    cfg = synth.config("oracle")
    a = synth.make_weights(cfg, np.random.default_rng(0), chunk_rows=1024)
    b = synth.make_weights(cfg, np.random.default_rng(0), chunk_rows=37)
    assert np.array_equal(a, b)


def test_levels_and_pmf():
    for name in synth.CONFIGS:
        cfg = synth.config(name)
        lv = synth.levels_of(cfg)
        assert lv.dtype == np.float32 and lv[cfg.k // 2] == 0.0 and len(lv) == cfg.k
        pmf = synth.pmf_of(cfg)
        assert abs(pmf.sum() - 1.0) < 1e-12 and pmf.min() > 0
        if cfg.pmf_kind == "conv-mode":
            assert pmf.argmax() == int(np.nonzero(lv == np.float32(0.01))[0][0])
        else:
            assert abs(pmf[cfg.k // 2] - cfg.p_zero) < 1e-12


def test_survey_probe_sizes_config1():
    """nnz 78,678; CER segments 6,910 (646 empty); CSER 6,264."""
    w, _ = synth.make_layer("oracle")
    cer, cser = numpy_port.encode_cer(w), numpy_port.encode_cser(w)
    assert len(cer["colI"]) == 78678
    assert len(cer["omegaPtr"]) - 1 == 6910
    assert int(np.sum(np.diff(cer["omegaPtr"]) == 0)) == 646
    assert len(cser["omegaPtr"]) - 1 == 6264


def test_survey_probe_nnz_config2():
    """SURVEY.md §8(a) table, config 2 (AlexNet fc6): nnz 3,395,269."""
    w = synth.make_weights(synth.config("alexnet-fc6"), np.random.default_rng(0))
    assert int(np.count_nonzero(w)) == 3395269


def test_device_generator_row_blocks_and_pmf():
    """make_weights_device: any row block equals the same rows of the full draw (row-sharded runs see
    one matrix), and the level frequencies follow the pmf."""
    torch = pytest.importorskip("torch")
    cfg = synth.config("oracle")
    full = synth.make_weights_device(cfg, 3, "cpu")
    part = synth.make_weights_device(cfg, 3, "cpu", row0=200, rows=250)
    assert torch.equal(full[200:450], part)
    assert not torch.equal(full, synth.make_weights_device(cfg, 4, "cpu"))
    vals, counts = np.unique(full.numpy(), return_counts=True)
    freq = dict(zip(vals.tolist(), (counts / full.numel()).tolist()))
    for v, p in zip(synth.levels_of(cfg).tolist(), synth.pmf_of(cfg)):
        assert abs(freq.get(v, 0.0) - p) < 5 * np.sqrt(p * (1 - p) / full.numel()) + 1e-4
