"""Batch sharding of independent series over ranks (BASELINE configs[4] on
G GPUs): the per-rank shares partition the batch into
contiguous, near-equal ranges -- every series runs exactly once, in order."""
from __future__ import annotations

import pytest

from paper_2511_10363_b200.distributed import batch_shard


@pytest.mark.parametrize("n", [0, 1, 7, 64, 65])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_batch_shard_partitions(n, world):
    shares = [batch_shard(n, r, world) for r in range(world)]
    flat = [i for s in shares for i in s]
    assert flat == list(range(n))
    sizes = [len(s) for s in shares]
    assert max(sizes) - min(sizes) <= 1
