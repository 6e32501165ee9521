"""CPU checks of the shared seeded-input / sampling helpers in workloads/ (no arithmetic of the
method lives there)."""
import workloads


def test_parity_points_cover_every_border():
    """The sampler itself: every border pixel of every image appears with every channel."""
    L = workloads.ConvLayer("t", 3, 8, 9, 7, 5, 3, 3, 1, 1)
    pts = workloads.parity_points(L, 9, 7, 100, seed=0)
    s = {tuple(v) for v in pts.tolist()}
    for n in range(3):
        for k in range(5):
            for p in range(9):
                for q in range(7):
                    if p in (0, 8) or q in (0, 6):
                        assert (n, k, p, q) in s
    inner = pts[-100:]
    assert ((inner[:, 2] > 0) & (inner[:, 2] < 8) & (inner[:, 3] > 0) & (inner[:, 3] < 6)).all()


def test_shard_range_partitions_the_batch():
    """N-split: contiguous shards, sizes within one, every image exactly once."""
    import pytest
    from paper_2008_04567_b200.nsplit import shard_range
    for n in (8, 9, 31, 32, 256):
        for world in (1, 2, 3, 4, 8):
            if n < world:
                continue
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert parts[-1][0] + parts[-1][1] == n
            sizes = [c for _, c in parts]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(256, 3, 8) == (96, 32)
    with pytest.raises(ValueError):
        shard_range(2, 0, 4)
    with pytest.raises(ValueError):
        shard_range(8, 8, 8)
