"""Host-side input helpers (workloads/): seeded generators and list orderings."""
import numpy as np
import pytest

from workloads import generate
from workloads.configs import CONFIGS
from workloads.gen import morton_sorted_cells, random_cells

torch = pytest.importorskip("torch")


def _morton_np(c, nx, ny):
    def spread(v):
        out = np.zeros_like(v)
        for b in range(21):
            out |= ((v >> b) & 1) << (3 * b)
        return out
    return spread(c % nx) | (spread((c // nx) % ny) << 1) | (spread(c // (nx * ny)) << 2)


@pytest.mark.parametrize("cells,c0,c1", [((5, 3, 2), 0, None), ((8, 8, 8), 64, 192), ((23, 17, 11), 391, 3519)])
def test_morton_sorted_cells(cells, c0, c1):
    got = morton_sorted_cells(cells, c0, c1).numpy()
    hi = int(np.prod(cells)) if c1 is None else c1
    assert sorted(got.tolist()) == list(range(c0, hi))          # a permutation of the range
    key = _morton_np(got, cells[0], cells[1])
    assert np.all(np.diff(key) > 0)                              # strictly increasing Morton code
    # every aligned 4^3 brick of a cube is one contiguous run of 64
    full = morton_sorted_cells((8, 8, 8)).numpy()
    bricks = (full % 8) // 4 + 2 * (((full // 8) % 8) // 4) + 4 * ((full // 64) // 4)
    assert all(len(set(bricks[i:i + 64])) == 1 for i in range(0, 512, 64))


def test_generators_are_seeded():
    for name in ("t1", "c2"):
        a, b = generate(name), generate(name)
        assert np.array_equal(a.X, b.X) and np.array_equal(a.y, b.y)
    r1, r2 = random_cells("t2", 100, 3), random_cells("t2", 100, 3)
    assert np.array_equal(r1, r2) and len(np.unique(r1)) == 100
    assert set(CONFIGS) >= {"c1", "c2", "c3", "c4", "c5"}
