"""The reference test-suite's deterministic RNG recipe (tests/oracles.hpp:39-50):
std::mt19937_64, doubles as ``(u64 >> 11) * 2**-53`` — never a library
distribution — plus its ``random_star_polygon`` fixture family
(tests/oracles.hpp:161-174).  Written from the published MT19937-64 algorithm
(Matsumoto & Nishimura, 2004)."""
from __future__ import annotations

import math

import numpy as np

_NN, _MM = 312, 156
_MATRIX_A = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)


class Rng:
    def __init__(self, seed: int):
        mt = [0] * _NN
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, _NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self._mt = np.array(mt, dtype=np.uint64)
        self._out = None
        self._pos = _NN

    def _twist(self):
        mt = self._mt
        one = np.uint64(1)

        def mix(upper, lower, far):
            x = (upper & _UM) | (lower & _LM)
            return far ^ (x >> one) ^ np.where((x & one) != 0, _MATRIX_A, np.uint64(0))

        a = mix(mt[0:_NN - _MM], mt[1:_NN - _MM + 1], mt[_MM:_NN])
        mt[0:_NN - _MM] = a
        b = mix(mt[_NN - _MM:_NN - 1], mt[_NN - _MM + 1:_NN], mt[0:_MM - 1])
        mt[_NN - _MM:_NN - 1] = b
        mt[_NN - 1] = mix(mt[_NN - 1:_NN], mt[0:1], mt[_MM - 1:_MM])[0]
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self._out = [int(v) for v in y]
        self._pos = 0

    def u64(self) -> int:
        if self._pos >= _NN:
            self._twist()
        v = self._out[self._pos]
        self._pos += 1
        return v

    def u01(self) -> float:
        return float(self.u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.u01()

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + self.u64() % (hi - lo + 1)


def random_star_polygon(rng: Rng, center_lat: float, center_lng: float, mean_radius_deg: float,
                        vertex_count: int) -> np.ndarray:
    """Strictly increasing vertex angles -> simple ring (oracles.hpp:161-174)."""
    pi = math.acos(-1.0)
    out = np.empty((vertex_count, 2))
    for i in range(vertex_count):
        angle = (i + 0.2 + 0.6 * rng.u01()) * 2.0 * pi / vertex_count
        radius = mean_radius_deg * rng.uniform(0.55, 1.45)
        out[i, 0] = center_lat + radius * math.sin(angle)
        out[i, 1] = center_lng + radius * math.cos(angle)
    return out


def random_points_in(rng: Rng, lat_lo, lat_hi, lng_lo, lng_hi, n: int) -> np.ndarray:
    """n x random_point_in (oracles.hpp:176-179): lat drawn before lng."""
    out = np.empty((n, 2))
    for i in range(n):
        out[i, 0] = rng.uniform(lat_lo, lat_hi)
        out[i, 1] = rng.uniform(lng_lo, lng_hi)
    return out
