"""Synthetic MNIST/Fashion-MNIST-shaped inputs and the angle encodings of the configs.

There is no network access for the real datasets, so the configs of BASELINE.json run on
synthetic images of the same shape:

  * MNIST-shaped: 10 class prototypes on 28x28 made of random blurred strokes (~19% ink);
    each sample is its class prototype shifted by up to +-2 px plus N(0, 0.1) noise on the ink,
    clipped to [0, 1]; balanced labels.
  * Fashion-shaped: filled blob silhouettes (~50% ink) with texture noise.

Encodings: configs 1/2 use PCA to 8/50 features followed by SPEC's min-max scaling to
[0, pi] with constant columns set to pi/2; the 784-qubit configs use the raw
pixels, angle = bw * pi * pixel.  Host-side numpy data preparation — not part of the hot path.
"""
from __future__ import annotations

import numpy as np

SIDE = 28
PIXELS = SIDE * SIDE


def _blur(img: np.ndarray, passes: int = 2) -> np.ndarray:
    k = np.array([0.25, 0.5, 0.25])
    out = img
    for _ in range(passes):
        out = np.apply_along_axis(lambda r: np.convolve(r, k, mode="same"), 1, out)
        out = np.apply_along_axis(lambda c: np.convolve(c, k, mode="same"), 0, out)
    return out


def _stroke_prototype(rng: np.random.Generator, ink: float = 0.19) -> np.ndarray:
    img = np.zeros((SIDE, SIDE))
    for _ in range(rng.integers(2, 4)):
        y, x = rng.uniform(6, 22, 2)
        ang = rng.uniform(0, 2 * np.pi)
        for _ in range(rng.integers(14, 26)):
            ang += rng.normal(0, 0.35)
            y = float(np.clip(y + np.sin(ang), 3, 24))
            x = float(np.clip(x + np.cos(ang), 3, 24))
            img[int(y), int(x)] = 1.0
    img = _blur(img, 2)
    thr = np.quantile(img, 1.0 - ink)
    return np.clip(img / max(thr, 1e-12), 0.0, 1.0) * (img >= 0.5 * thr)


def _silhouette_prototype(rng: np.random.Generator, ink: float = 0.5) -> np.ndarray:
    yy, xx = np.mgrid[0:SIDE, 0:SIDE]
    field = np.zeros((SIDE, SIDE))
    for _ in range(rng.integers(3, 6)):
        cy, cx = rng.uniform(7, 21, 2)
        sy, sx = rng.uniform(3, 8, 2)
        field += np.exp(-((yy - cy) ** 2 / (2 * sy * sy) + (xx - cx) ** 2 / (2 * sx * sx)))
    thr = np.quantile(field, 1.0 - ink)
    mask = field >= thr
    tex = 0.6 + 0.4 * _blur(rng.uniform(0, 1, (SIDE, SIDE)), 1)
    return np.clip(mask * tex, 0.0, 1.0)


def synthetic_images(n: int, kind: str = "mnist", seed: int = 0, classes: int = 10,
                     mix: float = 0.0):
    """(images [n, 784] in [0, 1], labels [n]) — balanced over `classes`.

    ``mix`` > 0 makes the classes overlap: sample k blends its class prototype with the
    prototype of another random class, weight m ~ U(0, mix) on the other one (m > 0.5 looks
    more like the other class), so a classifier cannot reach accuracy 1 (parity runs)."""
    rng = np.random.default_rng(seed)
    make = _stroke_prototype if kind == "mnist" else _silhouette_prototype
    protos = np.stack([make(rng) for _ in range(classes)])
    labels = np.arange(n) % classes
    rng.shuffle(labels)
    X = np.empty((n, PIXELS))
    shifts = rng.integers(-2, 3, size=(n, 2))
    if mix > 0:
        other = (labels + rng.integers(1, classes, n)) % classes
        weight = rng.uniform(0.0, mix, n)
    for k in range(n):
        base = protos[labels[k]]
        if mix > 0:
            base = (1.0 - weight[k]) * base + weight[k] * protos[other[k]]
        img = np.roll(base, tuple(shifts[k]), axis=(0, 1))
        ink = img > 0
        noise = rng.normal(0.0, 0.1, img.shape) * ink
        if kind != "mnist":
            noise += rng.normal(0.0, 0.05, img.shape) * ink
        X[k] = np.clip(img + noise, 0.0, 1.0).ravel()
    return X, labels


def pca_fit(X: np.ndarray, k: int):
    """Top-k principal axes of X (mean, components [k, d])."""
    mu = X.mean(axis=0)
    C = np.cov((X - mu).T)
    w, V = np.linalg.eigh(C)
    order = np.argsort(w)[::-1][:k]
    return mu, V[:, order].T


def pca_apply(X: np.ndarray, mu: np.ndarray, comps: np.ndarray) -> np.ndarray:
    return (X - mu) @ comps.T


def minmax_angles(train: np.ndarray, *others: np.ndarray):
    """SPEC.md:589-597 min-max to [0, pi] fitted on train; constant columns -> pi/2."""
    lo, hi = train.min(axis=0), train.max(axis=0)
    span = hi - lo
    const = span == 0

    def enc(A):
        out = np.where(const, np.pi / 2, (A - lo) / np.where(const, 1.0, span) * np.pi)
        return np.clip(out, 0.0, np.pi) if A is not train else out

    return (enc(train),) + tuple(enc(o) for o in others)


def pixel_angles(images: np.ndarray, bw: float = 1.0) -> np.ndarray:
    """784-qubit encoding: angle = bw * pi * pixel."""
    return bw * np.pi * images


def config_data(config_id: int, n_train: int, n_test: int, kind: str = "mnist",
                features: int | None = None, bw: float = 1.0, binary: tuple | None = None,
                classes: int = 10, mix: float = 0.0):
    """Angles for one config: seed = 240502630 + config_id."""
    seed = 240502630 + config_id
    if binary is not None:
        # balanced labels: the binary classes are len(binary)/classes of the draw
        draw = -(-(n_train + n_test) * classes // len(binary))
        X, y = synthetic_images(draw, kind, seed, classes, mix)
        keep = np.isin(y, binary)
        X, y = X[keep][: n_train + n_test], y[keep][: n_train + n_test]
        if len(y) < n_train + n_test:  # pragma: no cover - balanced draw always suffices
            raise ValueError("not enough samples of the binary classes")
    else:
        X, y = synthetic_images(n_train + n_test, kind, seed, classes, mix)
    Xtr, ytr, Xte, yte = X[:n_train], y[:n_train], X[n_train:], y[n_train:]
    if features is not None:
        mu, comps = pca_fit(Xtr, features)
        Atr, Ate = minmax_angles(pca_apply(Xtr, mu, comps), pca_apply(Xte, mu, comps))
    else:
        Atr, Ate = pixel_angles(Xtr, bw), pixel_angles(Xte, bw)
    return np.ascontiguousarray(Atr), ytr, np.ascontiguousarray(Ate), yte
