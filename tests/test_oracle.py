"""Pin the CPU oracles to the reference's own outputs (golden fixtures).

The fixtures were produced by running the reference (`lemt`) in the build
container (tests/golden/make_golden.py); these tests run anywhere.
"""

import numpy as np
import pytest

import recipes
from conftest import digest
from oracle import c_oracle, numpy_port

ORACLES = {"numpy": numpy_port, "c": c_oracle}


def _check_full(enc, g, kind):
    assert enc["omega"].tolist() == g["omega"]
    assert np.signbit(enc["omega"]).tolist() == g["omega_signbit"]
    assert enc["colI"].tolist() == g["colI"]
    assert enc["omegaPtr"].tolist() == g["omegaPtr"]
    assert enc["rowPtr"].tolist() == g["rowPtr"]
    assert enc["colI"].dtype.itemsize * 8 == g["bits"]["colI"]
    assert enc["omegaPtr"].dtype.itemsize * 8 == g["bits"]["omegaPtr"]
    assert enc["rowPtr"].dtype.itemsize * 8 == g["bits"]["rowPtr"]
    if kind == "cser":
        assert enc["omegaI"].tolist() == g["omegaI"]
        assert enc["omegaI"].dtype.itemsize * 8 == g["bits"]["omegaI"]
        assert enc["mode_index"] == g["mode_index"]


@pytest.mark.parametrize("oracle", sorted(ORACLES))
def test_small_cases_bit_exact(small_cases, oracle):
    mod = ORACLES[oracle]
    for case in small_cases:
        w = np.asarray(case["matrix"], dtype=float)
        x = np.asarray(case["x"], dtype=float)
        for kind in ("cer", "cser"):
            g = case[kind]
            encode = mod.encode_cer if kind == "cer" else mod.encode_cser
            if "error" in g:
                with pytest.raises(Exception) as err:
                    encode(w, index_bits=case["index_bits"], background=case["background"])
                assert type(err.value).__name__ == g["error"], case["name"]
                continue
            enc = encode(w, index_bits=case["index_bits"], background=case["background"])
            _check_full(enc, g, kind)
            y = mod.dot(enc, x)
            y_ref = np.asarray(g["y"], dtype=float)
            if oracle == "numpy":  # same evaluation order as the reference: bitwise
                assert np.array_equal(y, y_ref, equal_nan=True), case["name"]
            else:  # loop order: bitwise on integer data, else within 1e-12
                finite = np.isfinite(y_ref)
                assert np.array_equal(np.isfinite(y), finite)
                assert np.allclose(y[finite], y_ref[finite], rtol=1e-12, atol=1e-12), case["name"]


@pytest.mark.parametrize("oracle", sorted(ORACLES))
def test_recipe_families(recipe_digests, oracle):
    mod = ORACLES[oracle]
    for fam, cases in recipe_digests.items():
        for case in cases:
            w, x = recipes.RECIPES[fam](case["seed"])
            for kind in ("cer", "cser"):
                g = case[kind]
                enc = (mod.encode_cer if kind == "cer" else mod.encode_cser)(w)
                assert digest(enc["omega"]) == g["omega"], (fam, case["seed"])
                assert digest(enc["colI"]) == g["colI"]
                assert digest(enc["omegaPtr"]) == g["omegaPtr"]
                assert digest(enc["rowPtr"]) == g["rowPtr"]
                if kind == "cser":
                    assert digest(enc["omegaI"]) == g["omegaI"]
                    assert enc["mode_index"] == g["mode_index"]
                y = mod.dot(enc, x)
                if oracle == "numpy" or fam == "criterion3":
                    assert digest(y) == g["y_digest"], (fam, case["seed"], kind)


def test_c_oracle_configs(config_goldens):
    from paper_1805_10692_b200 import synth

    meta, ys = config_goldens
    for name in ("oracle", "resnet-conv", "alexnet-fc6"):
        w, _ = synth.make_layer(name)
        x1 = np.random.default_rng(1).standard_normal(w.shape[1], dtype=np.float32).astype(np.float64)
        for kind in ("cer", "cser"):
            enc = c_oracle.encode(w, kind)
            g = meta["configs"][name][kind]
            assert digest(enc["omega"]) == g["omega"]
            assert digest(enc["colI"]) == g["colI"]
            assert digest(enc["omegaPtr"]) == g["omegaPtr"]
            assert digest(enc["rowPtr"]) == g["rowPtr"]
            if kind == "cser":
                assert digest(enc["omegaI"]) == g["omegaI"]
            y = c_oracle.dot(enc, x1)
            y_ref = ys[f"{name}/{kind}/b1"]
            assert np.abs(y - y_ref).max() <= 1e-12 * np.abs(y_ref).max()


def test_numpy_port_config1_matrix_rhs(config_goldens):
    from paper_1805_10692_b200 import synth

    _, ys = config_goldens
    w, _ = synth.make_layer("oracle")
    xb = np.random.default_rng(2).standard_normal((w.shape[1], 8), dtype=np.float32).astype(np.float64)
    for kind in ("cer", "cser"):
        enc = numpy_port.encode_cer(w) if kind == "cer" else numpy_port.encode_cser(w)
        assert np.array_equal(numpy_port.dot(enc, xb), ys[f"oracle/{kind}/b8"])
        yc = c_oracle.dot(c_oracle.encode(w, kind), xb)
        assert np.abs(yc - ys[f"oracle/{kind}/b8"]).max() <= 1e-12 * np.abs(yc).max()


def test_row_block_slices_concatenate():
    from paper_1805_10692_b200 import synth

    w, xs = synth.make_layer("oracle")
    for encode in (numpy_port.encode_cer, numpy_port.encode_cser):
        enc = encode(w)
        full = c_oracle.dot(enc, xs[1])
        cuts = [0, 100, 101, 300, 512]
        parts = [c_oracle.dot(numpy_port.row_block(enc, a, b), xs[1]) for a, b in zip(cuts[:-1], cuts[1:])]
        assert np.array_equal(np.concatenate(parts), full)  # loop oracle is per-row: slicing is exact


def test_threaded_port_matches():
    from paper_1805_10692_b200 import synth

    w, xs = synth.make_layer("oracle")
    enc = numpy_port.encode_cer(w)
    y = numpy_port.dot(enc, xs[1])
    yt = numpy_port.dot_threaded(enc, xs[1], threads=4)
    assert np.abs(y - yt).max() <= 1e-12 * np.abs(y).max()


def test_empty_matrix_errors():
    for mod in ORACLES.values():
        with pytest.raises(IndexError):
            mod.encode_cer(np.zeros((0, 3)))
        with pytest.raises(IndexError):
            mod.encode_cser(np.zeros((2, 0)))


def test_dimension_mismatch_message():
    enc = numpy_port.encode_cer(np.eye(3))
    with pytest.raises(ValueError, match="mismatch"):
        numpy_port.dot(enc, np.ones(5))
    with pytest.raises(ValueError, match="mismatch"):
        c_oracle.dot(enc, np.ones(5))


def test_oracle_validate_decode_vs_reference_fixtures(validate_cases):
    """numpy_port.validate / decode against lemt.formats.validate / decode outcomes
    (tests/golden/make_validate_golden.py): same (array, offset, reason) for every corrupted encoding,
    same dense matrix (sha256) for every accepted one."""
    import hashlib

    from conftest import validate_case_arrays

    bases = validate_cases["bases"]
    for case in validate_cases["cases"]:
        enc = validate_case_arrays(bases, case)
        got = numpy_port.validate(enc)
        want = tuple(case["error"]) if case["error"] else None
        assert got == want, (case, got)
        if want is None:
            dense = numpy_port.decode(enc)
            assert hashlib.sha256(np.ascontiguousarray(dense).tobytes()).hexdigest() == case["decode_sha256"], case
