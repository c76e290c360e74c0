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


M128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _jump(state, inc, delta):
    """The LCG jump-ahead csrc/synth.cu uses (PCG paper), restated with Python integers."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, PCG_MULT, inc
    while delta:
        if delta & 1:
            acc_mult = acc_mult * cur_mult & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = (cur_mult + 1) * cur_plus & M128
        cur_mult = cur_mult * cur_mult & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


def _xsl_rr(state):
    x = (state >> 64) ^ (state & ((1 << 64) - 1))
    rot = state >> 122
    return ((x >> rot) | (x << (64 - rot))) & ((1 << 64) - 1)


def test_pcg64_restatement_matches_numpy():
    """The device generator's algorithm (csrc/synth.cu): element i of numpy's choice(K, p) is
    searchsorted(cdf, (xsl_rr(jump(s0, i + 1)) >> 11) * 2^-53, 'right'), including lane-strided jumps of 32."""
    cfg = synth.config("large")
    rng = np.random.default_rng(7)
    st = rng.bit_generator.state["state"]
    s0, inc = st["state"], st["inc"]
    draw = rng.choice(cfg.k, size=200, p=synth.pmf_of(cfg))
    cdf = synth.pmf_of(cfg).cumsum()
    cdf /= cdf[-1]
    for lane in (0, 5, 31):
        s = _jump(s0, inc, lane + 1)
        for e in range(lane, 200, 32):
            u = (_xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0)
            assert int(np.searchsorted(cdf, u, side="right")) == draw[e]
            s = _jump(s, inc, 32)
    # the inputs follow W in the draw order: the generator advanced past m*n draws
    a = synth.rng_after_weights(synth.config("oracle"), 3).standard_normal(5)
    r = np.random.default_rng(3)
    synth.make_weights(synth.config("oracle"), r)
    assert np.array_equal(a, r.standard_normal(5))
