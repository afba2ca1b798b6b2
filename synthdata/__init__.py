"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module is the ONLY code the oracle side (``oracle/``) and the product side
(``paper_1506_09067_b200/``) have in common.  It holds no arithmetic of the
method (no forward/backward/update): only the counter-based random-number
generator, the dataset recipes of BASELINE.json configs 0-4 and the parameter
initialiser, each a pure function of a seed.

Readings:

* PRNG: splitmix64.  Draw ``i`` (0-based) of a stream with seed ``s`` is
  ``mix(s + (i+1)*0x9E3779B97F4A7C15)`` -- counter based, so a whole stream is
  one vectorised numpy expression.
* uniform ``u = (x >> 40) * 2**-24`` in [0, 1) (24 bits, exact in fp32).
* Gaussian: Box-Muller on ``(1-u1, u2)``, cosine branch only (2 draws each).
* Config 0 (BASELINE.json configs[0]): per sample ``label = floor(10 u)`` then
  841 uniforms mapped to [-1, 1]; the test set continues the same stream.
* Configs 1-4 (configs[1..4]): 10 class prototypes (10 x 841 uniforms in
  [-1,1]) first; then per sample ``label = floor(10 u)`` and 841 Gaussians;
  pixel = clip(proto[label] + 0.5 * N(0,1), -1, 1).  Test set continues the
  stream after the training set (same prototypes).
* Parameters: U(-1/sqrt(fan_in), +1/sqrt(fan_in)) for W *and* b, drawn layer by
  layer, W then b, row-major in the normative flat layout, from the stream with
  seed ``data_seed ^ 0x5EED``.

All arrays are returned as float32 / int32 -- the bytes both sides consume.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
INIT_SEED_XOR = 0x5EED
IMG = 29 * 29  # 841 pixels, BASELINE.json configs[*] "input 1x29x29"


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws ``start .. start+count-1`` of the splitmix64 stream ``seed``."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + 1 + count, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, start: int, count: int) -> np.ndarray:
    """u = (x >> 40) * 2^-24 in [0, 1), float64 (exactly representable in fp32)."""
    return (splitmix64(seed, start, count) >> np.uint64(40)).astype(np.float64) * (2.0 ** -24)


def _gauss_from_pairs(u: np.ndarray) -> np.ndarray:
    """Box-Muller, cosine branch, on consecutive (u1, u2) pairs."""
    u1 = u[0::2]
    u2 = u[1::2]
    return np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * np.pi * u2)


@dataclass
class Dataset:
    x_train: np.ndarray  # float32 [n][841]
    y_train: np.ndarray  # int32 [n]
    x_test: np.ndarray
    y_test: np.ndarray

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.x_train, self.y_train, self.x_test, self.y_test):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


def uniform_dataset(seed: int, n_train: int, n_test: int) -> Dataset:
    """Config 0 recipe: label = floor(10u), then 841 uniforms in [-1, 1]."""
    per = 1 + IMG
    n = n_train + n_test
    u = uniform01(seed, 0, n * per).reshape(n, per)
    y = np.minimum(np.floor(u[:, 0] * 10.0), 9).astype(np.int32)
    x = (2.0 * u[:, 1:] - 1.0).astype(np.float32)
    return Dataset(x[:n_train].copy(), y[:n_train].copy(), x[n_train:].copy(), y[n_train:].copy())


def prototype_samples(seed: int, first: int, count: int) -> tuple[np.ndarray, np.ndarray]:
    """Samples ``first .. first+count-1`` of the prototype+noise stream (configs 1-4).

    Sample j consumes draws [10*841 + j*(1+2*841), ...): one label draw then 841
    Box-Muller pairs.  Chunked so 480k-sample sets fit in memory.
    """
    protos = (2.0 * uniform01(seed, 0, 10 * IMG) - 1.0).reshape(10, IMG)
    per = 1 + 2 * IMG
    base = 10 * IMG
    xs = np.empty((count, IMG), dtype=np.float32)
    ys = np.empty((count,), dtype=np.int32)
    chunk = 4096
    for c0 in range(0, count, chunk):
        c = min(chunk, count - c0)
        u = uniform01(seed, base + (first + c0) * per, c * per).reshape(c, per)
        lab = np.minimum(np.floor(u[:, 0] * 10.0), 9).astype(np.int32)
        g = _gauss_from_pairs(u[:, 1:].reshape(-1)).reshape(c, IMG)
        xs[c0:c0 + c] = np.clip(protos[lab] + 0.5 * g, -1.0, 1.0).astype(np.float32)
        ys[c0:c0 + c] = lab
    return xs, ys


def prototype_dataset(seed: int, n_train: int, n_test: int) -> Dataset:
    xtr, ytr = prototype_samples(seed, 0, n_train)
    xte, yte = prototype_samples(seed, n_train, n_test)
    return Dataset(xtr, ytr, xte, yte)


def init_params(data_seed: int, blocks) -> np.ndarray:
    """Initial parameters in the normative flat layout.

    ``blocks`` = iterable of ``(fan_in, n_weights, n_bias)`` per weighted layer,
    in layer order (the caller owns the shape chain).  W and b of a layer are
    both U(-a, a), a = 1/sqrt(fan_in), drawn W first then b.
    """
    seed = data_seed ^ INIT_SEED_XOR
    out = []
    pos = 0
    for fan_in, nw, nb in blocks:
        a = 1.0 / np.sqrt(float(fan_in))
        u = uniform01(seed, pos, nw + nb)
        pos += nw + nb
        out.append(((2.0 * u - 1.0) * a).astype(np.float32))
    return np.concatenate(out) if out else np.zeros(0, np.float32)


# ---------------------------------------------------------------------------
# Workloads of BASELINE.json (architectures are configuration, not arithmetic)
# Layer tuple: (kind, units, kernel, act); kind 1=conv 2=maxpool 3=full,
# act 0=tanh 1=identity (the last FULL layer gives the logits).
# ---------------------------------------------------------------------------
CONV, POOL, FULL = 1, 2, 3
TANH, IDENT = 0, 1

ARCHS = {
    # configs[0], configs[1]: conv 5 maps 4x4, tanh, 2x2 max-pool, FC 845->10
    "tiny": [(CONV, 5, 4, TANH), (POOL, 0, 2, TANH), (FULL, 10, 0, IDENT)],
    # configs[2] (= Table I medium)
    "medium": [(CONV, 20, 4, TANH), (POOL, 0, 2, TANH), (CONV, 40, 5, TANH), (POOL, 0, 3, TANH),
               (FULL, 150, 0, TANH), (FULL, 10, 0, IDENT)],
    # configs[3], configs[4]
    "large": [(CONV, 20, 4, TANH), (POOL, 0, 2, TANH), (CONV, 60, 3, TANH), (POOL, 0, 2, TANH),
              (CONV, 100, 2, TANH), (POOL, 0, 2, TANH), (FULL, 150, 0, TANH), (FULL, 10, 0, IDENT)],
    # Table I small / large of the paper (NEXT-1 only)
    "paper_small": [(CONV, 5, 4, TANH), (POOL, 0, 2, TANH), (CONV, 10, 5, TANH), (POOL, 0, 3, TANH),
                    (FULL, 50, 0, TANH), (FULL, 10, 0, IDENT)],
    "paper_large": [(CONV, 20, 4, TANH), (POOL, 0, 1, TANH), (CONV, 60, 5, TANH), (POOL, 0, 2, TANH),
                    (CONV, 100, 6, TANH), (POOL, 0, 2, TANH), (FULL, 150, 0, TANH), (FULL, 10, 0, IDENT)],
}


@dataclass(frozen=True)
class Workload:
    name: str
    arch: str
    data: str  # "uniform" | "prototype"
    seed: int
    n_train: int
    n_test: int
    lr0: float
    epochs: int
    sync_batch: int


WORKLOADS = {
    "config0": Workload("config0", "tiny", "uniform", 0, 1000, 200, 0.01, 1, 1),
    "config1": Workload("config1", "tiny", "prototype", 1, 60000, 10000, 0.001, 15, 64),
    "config2": Workload("config2", "medium", "prototype", 1, 60000, 10000, 0.001, 15, 64),
    "config3": Workload("config3", "large", "prototype", 1, 60000, 10000, 0.001, 15, 64),
    "config4": Workload("config4", "large", "prototype", 2, 480000, 10000, 0.001, 15, 64),
}


def make_dataset(w: Workload, n_train: int | None = None, n_test: int | None = None) -> Dataset:
    ntr = w.n_train if n_train is None else n_train
    nte = w.n_test if n_test is None else n_test
    if w.data == "uniform":
        if ntr != w.n_train:
            # the test set continues the stream after the FULL training set
            full = uniform_dataset(w.seed, w.n_train, nte)
            return Dataset(full.x_train[:ntr], full.y_train[:ntr], full.x_test, full.y_test)
        return uniform_dataset(w.seed, ntr, nte)
    xtr, ytr = prototype_samples(w.seed, 0, ntr)
    xte, yte = prototype_samples(w.seed, w.n_train, nte)
    return Dataset(xtr, ytr, xte, yte)
