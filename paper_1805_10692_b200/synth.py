"""Seeded synthetic layers standing in for the paper's pretrained weights.

The reference ships no generator and its experiments used pretrained
AlexNet/VGG16/ResNet152 layers that are not available here
(``PAPER.md:460-464``).  These are the build's definition of the five
BASELINE.json configs:

* ``rng = np.random.default_rng(seed)`` (seed 0); W is drawn first, then
  each X in the listed batch order; B=1 is column 0 of its own (n, 1) draw.
* codebook ``levels = (arange(K) - K//2) * (R / (K//2))`` in float64, cast
  to float32, so ``levels[K//2] == 0`` exactly.
* ``W = levels[rng.choice(K, size=(m, n), p=pmf)]`` (fp32, row-major).
* ``X = rng.standard_normal((n, B), dtype=float32)``, optionally ReLU'd.
* non-zero levels are ranked by ``(|v|, v)`` for the pmf shapes.

W is generated in row chunks; ``Generator.choice`` with ``p`` draws one
uniform per element in row-major order, so chunked draws equal one call
(``tests/test_synth.py`` checks this).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["LayerConfig", "CONFIGS", "config", "levels_of", "pmf_of", "make_weights", "make_inputs"]


@dataclass(frozen=True)
class LayerConfig:
    name: str
    m: int
    n: int
    k: int
    radius: float
    pmf_kind: str  # "geometric" | "laplace" | "zipf" | "conv-mode"
    p_zero: float
    batches: tuple[int, ...]
    relu: bool
    shape_param: float = 0.0  # ratio / scale / exponent of the non-zero pmf
    description: str = ""


CONFIGS: dict[str, LayerConfig] = {
    "oracle": LayerConfig(
        "oracle", 512, 1024, 16, 1.0, "geometric", 0.85, (1,), False, 0.7,
        "CPU-runnable oracle: 16-level codebook on [-1,1], 85% zeros, geometric(0.7)",
    ),
    "alexnet-fc6": LayerConfig(
        "alexnet-fc6", 4096, 9216, 128, 0.05, "laplace", 0.91, (1, 64), False, 0.0125,
        "AlexNet-fc6-shaped: 128 levels on [-0.05,0.05], 91% zeros, Laplace-weighted",
    ),
    "vgg-fc6": LayerConfig(
        "vgg-fc6", 4096, 25088, 32, 0.05, "zipf", 0.96, (128,), True, 1.2,
        "VGG16-fc6-shaped: 32 levels, 96% zeros, Zipf(1.2); X = ReLU(N(0,1))",
    ),
    "resnet-conv": LayerConfig(
        "resnet-conv", 512, 4608, 16, 0.08, "conv-mode", 0.40, (1568,), True, 0.7,
        "ResNet-152 3x3 conv as im2col: mode 0.01 at 45%, 40% zeros; X = ReLU(N(0,1))",
    ),
    "large": LayerConfig(
        "large", 32768, 32768, 256, 0.2, "laplace", 0.70, (256,), False, 0.02,
        "Large low-entropy layer: 256 levels, quantised Laplace(0,0.02), 70% zeros",
    ),
}

_ALIASES = {"1": "oracle", "2": "alexnet-fc6", "3": "vgg-fc6", "4": "resnet-conv", "5": "large"}


def config(name: str | int) -> LayerConfig:
    key = _ALIASES.get(str(name), str(name))
    if key not in CONFIGS:
        raise KeyError(f"unknown config {name!r}; known: {sorted(CONFIGS)}")
    return CONFIGS[key]


def levels_of(cfg: LayerConfig) -> np.ndarray:
    half = cfg.k // 2
    return ((np.arange(cfg.k) - half) * (cfg.radius / half)).astype(np.float32)


def pmf_of(cfg: LayerConfig) -> np.ndarray:
    lv = levels_of(cfg).astype(np.float64)
    zero = cfg.k // 2
    pmf = np.zeros(cfg.k)
    pmf[zero] = cfg.p_zero
    others = [i for i in range(cfg.k) if i != zero]
    if cfg.pmf_kind == "conv-mode":
        mode = int(np.nonzero(levels_of(cfg) == np.float32(0.01))[0][0])
        pmf[mode] = 0.45
        others = [i for i in others if i != mode]
        rest = 1.0 - cfg.p_zero - 0.45
    else:
        rest = 1.0 - cfg.p_zero
    order = sorted(others, key=lambda i: (abs(lv[i]), lv[i]))
    j = np.arange(1, len(order) + 1, dtype=np.float64)
    if cfg.pmf_kind in ("geometric", "conv-mode"):
        w = cfg.shape_param ** (j - 1)
    elif cfg.pmf_kind == "laplace":
        w = np.exp(-np.abs(lv[order]) / cfg.shape_param)
    elif cfg.pmf_kind == "zipf":
        w = j ** (-cfg.shape_param)
    else:  # pragma: no cover - closed set above
        raise ValueError(cfg.pmf_kind)
    pmf[order] = rest * w / w.sum()
    return pmf / pmf.sum()


def make_weights(cfg: LayerConfig, rng: np.random.Generator, rows: int | None = None,
                 chunk_rows: int = 1024) -> np.ndarray:
    """W (fp32, m x n) drawn first from ``rng``; ``rows`` limits to a leading row slice."""
    m = cfg.m if rows is None else int(rows)
    lv = levels_of(cfg)
    pmf = pmf_of(cfg)
    out = np.empty((m, cfg.n), dtype=np.float32)
    for r0 in range(0, m, chunk_rows):
        r1 = min(m, r0 + chunk_rows)
        out[r0:r1] = lv[rng.choice(cfg.k, size=(r1 - r0, cfg.n), p=pmf)]
    return out


def _pcg64_words(rng: np.random.Generator):
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("the device draw reproduces numpy's PCG64 generator only")
    s, inc = st["state"]["state"], st["state"]["inc"]
    mask = (1 << 64) - 1
    return (np.array([s & mask, s >> 64], dtype=np.uint64), np.array([inc & mask, inc >> 64], dtype=np.uint64))


def make_weights_device(cfg: LayerConfig, seed: int, device, row0: int = 0, rows: int | None = None):
    """Rows [row0, row0 + rows) of a config's W drawn ON THE DEVICE, bit-identical to ``make_weights`` with
    ``np.random.default_rng(seed)`` (W is the first draw of the seeded generator): the
    library's PCG64 kernel (cerdot_synth_choice) jumps to element row0 * n and reproduces numpy's
    ``choice(K, p=pmf)``.  Used for the 32768^2 config, whose numpy draw takes about a minute on the host;
    any row block is the same rows of the one seeded matrix, whichever shard draws it."""
    import torch

    from . import _native

    m = cfg.m - row0 if rows is None else int(rows)
    state, inc = _pcg64_words(np.random.default_rng(seed))
    pmf = pmf_of(cfg)
    cdf = pmf.cumsum()
    cdf /= cdf[-1]
    dev = torch.device(device)
    cdf_d = torch.from_numpy(cdf).to(dev)
    lv_d = torch.from_numpy(levels_of(cfg)).to(dev)
    out = torch.empty((m, cfg.n), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _native.check(_native.lib().cerdot_synth_choice(
            state.ctypes.data, inc.ctypes.data, int(row0) * cfg.n, cdf_d.data_ptr(), lv_d.data_ptr(), cfg.k,
            m * cfg.n, out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
        torch.cuda.current_stream(dev).synchronize()  # state / inc are host arrays read at launch
    return out


def rng_after_weights(cfg: LayerConfig, seed: int) -> np.random.Generator:
    """The seeded generator positioned after W's m * n draws (for the inputs, drawn next in §8(d)'s order)."""
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance(cfg.m * cfg.n)
    return rng


def make_inputs(cfg: LayerConfig, rng: np.random.Generator, batch: int) -> np.ndarray:
    """One X draw (fp32, n x B, row-major); B=1 returns the (n,) vector of column 0."""
    x = rng.standard_normal((cfg.n, batch), dtype=np.float32)
    if cfg.relu:
        np.maximum(x, 0.0, out=x)
    return np.ascontiguousarray(x[:, 0]) if batch == 1 else x


def input_for(cfg: LayerConfig, seed: int, batch: int) -> np.ndarray:
    """X of a listed batch in §8(d)'s order (drawn after W, batches in the listed order); B=1 when the
    config does not list it: column 0 of the first listed batch's draw."""
    rng = rng_after_weights(cfg, seed)
    first = None
    for b in cfg.batches:
        x = make_inputs(cfg, rng, b)
        if b == batch:
            return x
        if first is None:
            first = x
    if batch == 1:
        return np.ascontiguousarray(first[:, 0])
    raise ValueError(f"batch {batch} is not listed for config {cfg.name} ({cfg.batches})")


def make_layer(cfg: LayerConfig | str, seed: int = 0, rows: int | None = None):
    """(W, {B: X}) for a config, drawn in the documented order."""
    if not isinstance(cfg, LayerConfig):
        cfg = config(cfg)
    rng = np.random.default_rng(seed)
    w = make_weights(cfg, rng, rows=rows)
    xs = {b: make_inputs(cfg, rng, b) for b in cfg.batches}
    return w, xs
