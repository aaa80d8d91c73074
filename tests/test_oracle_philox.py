"""Pins the oracle's Philox4x32-10 and its uniform mapping (reading R2) -- CPU only."""
import numpy as np
import pytest

from tests.philox_tool import curand_philox

# Published Philox4x32-10 known-answer vectors (Salmon, Moraes, Dror, Shaw, SC'11,
# Random123 kat_vectors): (counter, key) -> output.
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_published_kat(oracle_mod):
    for ctr, key, want in KAT:
        assert oracle_mod.philox4x32_10(ctr, key) == want


def test_against_curand(oracle_mod):
    rng = np.random.default_rng(123)
    rows = [tuple(int(v) for v in rng.integers(0, 2**32, 6, dtype=np.uint64)) for _ in range(300)]
    rows += [(j, 0, b, 0, 0, 0) for j in range(20) for b in range(3)]
    rows += [(j, 0, 1023, 0, 0xDEADBEEF, 0x01234567) for j in range(0, 70000, 4999)]
    ref = curand_philox(rows)
    for r, want in zip(rows, ref):
        assert oracle_mod.philox4x32_10(r[:4], r[4:]) == want


def test_uniform_mapping_exact(oracle_mod):
    """u = (2 (x >> 12) + 1) 2^-53 with x = (r.y << 32) | r.x from curand's output."""
    seeds = [0, 1, 0x123456789ABCDEF0]
    rows, keys = [], []
    for seed in seeds:
        for j in [0, 1, 2, 255, 3119, 16383, 65535, 2**33 + 5]:
            for b in [0, 1, 1023, 2**40 + 3]:
                rows.append((j & 0xFFFFFFFF, j >> 32, b & 0xFFFFFFFF, b >> 32,
                             seed & 0xFFFFFFFF, seed >> 32))
                keys.append((seed, j, b))
    ref = curand_philox(rows)
    for (seed, j, b), r in zip(keys, ref):
        x = (r[1] << 32) | r[0]
        want = (2 * (x >> 12) + 1) / 2.0**53
        u = oracle_mod.uniform(seed, j, b)
        assert u == want
        assert 0.0 < u < 1.0
        m = u * 2.0**53
        assert m == int(m) and int(m) % 2 == 1


def test_uniform_moments(oracle_mod):
    u = np.array([oracle_mod.uniform(7, j, 0) for j in range(20000)])
    assert abs(u.mean() - 0.5) < 4 * np.sqrt(1 / 12 / len(u))
    assert abs((u ** 2).mean() - 1 / 3) < 0.01
