"""splitmix64 stream used for restart vectors (testprob.py:26-38 semantics).

Restated so restart vectors are bit-identical to the reference's:
z_i = seed + i * 0x9E3779B97F4A7C15 (i = 1..count), then the splitmix64
finaliser; uniforms in (0, 1] are ((z >> 11) + 1) * 2**-53.
"""

from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, count):
    i = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(int(seed) % (1 << 64)) + i * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform_open_closed(seed, count):
    return ((splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
