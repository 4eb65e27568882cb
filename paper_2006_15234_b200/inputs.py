"""Seeded synthetic workloads for the BASELINE configs (host side, numpy).

The reference has no Gaussian sampler, so the harness defines one:
Box-Muller over the reference's SplitMix64 stream (proj/include/peps/rng.hpp:12-32).
The same host arrays are fed to the GPU library and to the oracle, so the
generator itself only has to be deterministic, not bit-identical to anything.

Layouts follow the reference: PEPS site tensors are (phys, up, left, down, right)
with lattice-edge bonds of extent 1 (proj/src/state.cpp:22-42); boundary MPS
sites are (pb*pk, left, right) (proj/src/contraction.cpp:254-267).
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
_G = np.uint64(GAMMA)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def splitmix_stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Outputs start..start+n-1 of SplitMix64(seed) (rng.hpp:17-23)."""
    i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(np.uint64(seed & MASK) + i * _G)


def unit(u: np.ndarray) -> np.ndarray:
    """rng.hpp:26: (x >> 11) * 2^-53, uniform on [0, 1)."""
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _mix_int(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def derive_seed(base: int, *parts: int) -> int:
    """rng.hpp:38-44: chain of SplitMix64(base ^ (part + gamma)).next_u64()."""
    s = base & MASK
    for p in parts:
        st = (s ^ ((p + GAMMA) & MASK)) & MASK
        s = _mix_int((st + GAMMA) & MASK)
    return s


def gaussian(shape, seed: int, scale: float = 1.0) -> np.ndarray:
    """iid N(0, scale^2) real entries, stored complex128 with zero imaginary part.

    Box-Muller on consecutive SplitMix64 pairs: z0 = r cos(2 pi u2), z1 = r sin(2 pi u2),
    r = sqrt(-2 log(1 - u1)).
    """
    n = int(np.prod(shape)) if len(shape) else 1
    npair = (n + 1) // 2
    u = unit(splitmix_stream(seed, 2 * npair))
    u1, u2 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log1p(-u1))
    z = np.empty(2 * npair)
    z[0::2] = r * np.cos(2.0 * np.pi * u2)
    z[1::2] = r * np.sin(2.0 * np.pi * u2)
    return (z[:n] * scale).astype(np.complex128).reshape(shape)


def peps_site_shape(rows, cols, r, c, bond, d=2):
    return (d, 1 if r == 0 else bond, 1 if c == 0 else bond, 1 if r == rows - 1 else bond,
            1 if c == cols - 1 else bond)


def random_peps(rows: int, cols: int, bond: int, seed: int, d: int = 2, scale: float = 1.0):
    """Gaussian PEPS; site (r, c) uses seed derive_seed(seed, r, c)."""
    return [gaussian(peps_site_shape(rows, cols, r, c, bond, d), derive_seed(seed, r, c), scale)
            for r in range(rows) for c in range(cols)]


def random_boundary(length: int, phys: tuple, m: int, seed: int, scale: float = 1.0):
    """Gaussian two-layer boundary MPS: sites (pb*pk, left, right), bonds m, edges 1."""
    pb, pk = phys
    sites = []
    for c in range(length):
        shape = (pb * pk, 1 if c == 0 else m, 1 if c == length - 1 else m)
        sites.append(gaussian(shape, derive_seed(seed, 0xB0, c), scale))
    return sites, [(pb, pk)] * length


# --------------------------------------------------------------------------- BASELINE configs

def config1(seed: int = 1):
    """4x4, d=2, r=2, N(0,1); m=4, oversample 4, q=1."""
    return dict(rows=4, cols=4, d=2, sites=random_peps(4, 4, 2, seed), m=4, oversample=4,
                power_iters=1, seed=seed)


def config2(seed: int = 2, length: int = 8, bond: int = 8, m: int = 64):
    """Standalone row absorb: boundary L=8, m=64 N(0,1) + one interior row (3-row state, row=1)."""
    sites = random_peps(3, length, bond, seed)
    top, phys = random_boundary(length, (bond, bond), m, derive_seed(seed, 0x70))
    return dict(rows=3, cols=length, d=2, sites=sites, top=top, phys=phys, row=1, m=m,
                oversample=8, power_iters=2, seed=seed)


def config3(seed: int = 3, n: int = 16, bond: int = 6, m: int = 36):
    """16x16, r=6, N(0,1)/sqrt(r^2 d); m=36; defaults q=2, oversample=-1 (-> 5)."""
    scale = 1.0 / np.sqrt(bond * bond * 2)
    return dict(rows=n, cols=n, d=2, sites=random_peps(n, n, bond, seed, scale=scale), m=m,
                oversample=-1, power_iters=2, seed=seed)


def config5(seed: int = 5, n: int = 32, bond: int = 8, m: int = 64):
    """32x32, r=8, N(0,1)/sqrt(128); m=64; q=2, oversample=8 (stated choice)."""
    scale = 1.0 / np.sqrt(bond * bond * 2)
    return dict(rows=n, cols=n, d=2, sites=random_peps(n, n, bond, seed, scale=scale), m=m,
                oversample=8, power_iters=2, seed=seed)
