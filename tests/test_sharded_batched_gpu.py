"""C5-style system sharding (north-star (5)): rank r of N solves its own
contiguous block of systems with no communication; the union over ranks is
bit-identical to one device solving the whole batch.  Ranks are solved one
after the other on this GPU (no kernel waits on another rank)."""

import numpy as np
import pytest

from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu


class _RankOnly:
    """comm stand-in for rank `rank` of `world` (no collective is issued without gather)."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world


@pytest.mark.parametrize("world", [2, 3, 8])
def test_system_shards_union_equals_whole_batch(world):
    import paper_2104_12570_b200 as pb
    from paper_2104_12570_b200.sharded import partition_systems, solve_bak_batched_sharded
    nsys = 37
    xs = np.stack([orc.config_c5_system(s)[0] for s in range(nsys)])
    ys = np.stack([orc.config_c5_system(s)[1] for s in range(nsys)])
    cfg = pb.SolveConfig(max_iter=60, tol=0)
    whole = pb.solve_bak_batched(xs, ys, cfg)
    seen = []
    for r in range(world):
        s0, s1, rep = solve_bak_batched_sharded(xs, ys, cfg, _RankOnly(r, world))
        assert (s0, s1) == partition_systems(nsys, world, r)
        assert np.array_equal(rep.a_hat, whole.a_hat[s0:s1])
        assert np.array_equal(rep.residual, whole.residual[s0:s1])
        assert np.array_equal(rep.sweeps_run, whole.sweeps_run[s0:s1])
        seen.extend(range(s0, s1))
    assert seen == list(range(nsys))
    for s in (0, nsys - 1):
        ref = orc.solve(xs[s], ys[s], max_iter=60, tol=0)
        assert orc.rel_coeff_err(whole.a_hat[s], ref["a_hat"]) <= 1e-4


def test_system_shards_local_input():
    import paper_2104_12570_b200 as pb
    from paper_2104_12570_b200.sharded import partition_systems, solve_bak_batched_sharded
    nsys, world = 20, 2
    xs = np.stack([orc.config_c5_system(s)[0] for s in range(nsys)])
    ys = np.stack([orc.config_c5_system(s)[1] for s in range(nsys)])
    cfg = pb.SolveConfig(max_iter=30, tol=0)
    whole = pb.solve_bak_batched(xs, ys, cfg)
    for r in range(world):
        a, b = partition_systems(nsys, world, r)
        s0, s1, rep = solve_bak_batched_sharded(xs[a:b], ys[a:b], cfg, _RankOnly(r, world), local=True)
        assert np.array_equal(rep.a_hat, whole.a_hat[a:b])
