"""Seeded synthetic grayscale images (the stand-ins for the paper's test images).

The paper measures on "well-known images" (Lena, Baboon, F16; §4)
which are not available here.  BASELINE.json `configs` fixes only the ingredients of the
generator ("sum of 3 random-frequency sinusoids + 4 random axis-aligned rectangles of
constant intensity + Gaussian noise sigma=4, clipped to [0,255]", plus "a 1/f-spectrum
texture layer" for the 512x512 config).  The concrete distributions are the reading
recorded in DESIGN.md §"Input recipe".

This module is shared by the oracle (oracle/) and the CUDA path (paper_1501_04140_b200/)
and therefore holds NONE of the method's arithmetic: it only draws pixels.
"""
from __future__ import annotations

import numpy as np


def make_image(N: int, seed: int, texture: bool = False) -> np.ndarray:
    """Return an N x N uint8 image, row-major, pixel (x, y) = img[y, x].

    Draw order (fixed, from numpy.random.Generator(PCG64(seed))):
      1. three sinusoids, each: A ~ U[16,48], f ~ U[1/64,1/8] cycles/px,
         theta ~ U[0,pi), phi ~ U[0,2pi)
      2. four rectangles, each: c ~ U[-64,64], w ~ U{N/16..N/4}, h ~ U{N/16..N/4},
         x0 ~ U{0..N-w}, y0 ~ U{0..N-h}
      3. (texture only) white N(0,1) field N x N, shaped by 1/|f| in the Fourier domain
         (DC = 0) and rescaled to standard deviation 12
      4. per-pixel noise N(0, 4^2)
    then rint (half-even), clip to [0,255], cast to uint8.
    """
    if N < 1:
        raise ValueError("N must be positive")
    rng = np.random.Generator(np.random.PCG64(seed))
    y, x = np.mgrid[0:N, 0:N].astype(np.float64)
    img = np.full((N, N), 128.0)
    for _ in range(3):
        A = rng.uniform(16.0, 48.0)
        f = rng.uniform(1.0 / 64.0, 1.0 / 8.0)
        th = rng.uniform(0.0, np.pi)
        ph = rng.uniform(0.0, 2.0 * np.pi)
        img += A * np.sin(2.0 * np.pi * f * (x * np.cos(th) + y * np.sin(th)) + ph)
    lo, hi = max(1, N // 16), max(1, N // 4)
    for _ in range(4):
        c = rng.uniform(-64.0, 64.0)
        w = int(rng.integers(lo, hi, endpoint=True))
        h = int(rng.integers(lo, hi, endpoint=True))
        x0 = int(rng.integers(0, N - w, endpoint=True))
        y0 = int(rng.integers(0, N - h, endpoint=True))
        img[y0:y0 + h, x0:x0 + w] += c
    if texture:
        white = rng.standard_normal((N, N))
        F = np.fft.fft2(white)
        fy = np.fft.fftfreq(N)[:, None]
        fx = np.fft.fftfreq(N)[None, :]
        mag = np.sqrt(fx * fx + fy * fy)
        mag[0, 0] = np.inf  # DC -> 0
        tex = np.real(np.fft.ifft2(F / mag))
        sd = tex.std()
        if sd > 0:
            img += tex * (12.0 / sd)
    img += rng.normal(0.0, 4.0, size=(N, N))
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def ramp_image(N: int) -> np.ndarray:
    """I(x, y) = x + y (requires 2N-2 <= 255).  Zero-error fixture (SURVEY.md §8(c) pins)."""
    if 2 * N - 2 > 255:
        raise ValueError("ramp needs 2N-2 <= 255")
    y, x = np.mgrid[0:N, 0:N]
    return (x + y).astype(np.uint8)


def constant_image(N: int, value: int = 77) -> np.ndarray:
    return np.full((N, N), value, dtype=np.uint8)


def random_image(N: int, seed: int, lo: int = 0, hi: int = 255) -> np.ndarray:
    """Uniform i.i.d. pixels; used for edge-case and brute-force tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(lo, hi, size=(N, N), endpoint=True).astype(np.uint8)


def sample_indices(n: int, k: int, seed: int) -> np.ndarray:
    """k distinct sorted indices out of range(n) (seeded).  Used to pick sampled outputs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    k = min(k, n)
    return np.sort(rng.choice(n, size=k, replace=False)).astype(np.int64)
