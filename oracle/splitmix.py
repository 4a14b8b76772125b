"""SplitMix64 and the reference's synthetic input generator, vectorised.

TEST INFRASTRUCTURE (oracle/).  Restates pipec::SplitMix64
(proj/include/pipec/common.hpp:74-97) and random_tensor / load_inputs
(proj/include/pipec/cli.hpp:41-71): element i of a tensor seeded with `seed`
is range(-8, 8) of the (i+1)-th draw.  Pinned against the compiled reference
in tests/test_oracle.py.
"""
import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix_draws(seed: int, count: int) -> np.ndarray:
    """The first `count` outputs of SplitMix64(seed).next() (common.hpp:77-82)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def random_tensor(count: int, seed: int, lo: int = -8, hi: int = 8) -> np.ndarray:
    """cli.hpp:41-46: ints in [lo, hi] via range() = lo + next() % (hi-lo+1)."""
    n = np.uint64(hi - lo + 1)
    return (splitmix_draws(seed, count) % n).astype(np.int64) + lo


def uniform_tensor(count: int, seed: int) -> np.ndarray:
    """D-float inputs: uniform() in [0,1) (common.hpp:89) mapped to [-1, 1)."""
    u = (splitmix_draws(seed, count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def gemm_inputs(M, N, K, batch=1, seed=0, trial=None):
    """Inputs exactly as the reference binds them: A gets seed+0, B seed+1
    (load_inputs, cli.hpp:66; verify uses seed + 1000003*t + which, cli.hpp:295)."""
    base = seed if trial is None else seed + 1000003 * trial
    a = random_tensor(batch * M * K, base + 0)
    b = random_tensor(batch * K * N, base + 1)
    shp_a = (batch, M, K) if batch > 1 else (M, K)
    shp_b = (batch, K, N) if batch > 1 else (K, N)
    return a.reshape(shp_a), b.reshape(shp_b)
