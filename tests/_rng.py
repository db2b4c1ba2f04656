"""splitmix64 -> uniform(-1, 1), bit-identical to SplitMix in oracle/ref_driver.cpp.

Test infrastructure: generates the seeded random grid functions of the parity tests.
"""
import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """Draws number start .. start+count-1 of the stream seeded with `seed`."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0
