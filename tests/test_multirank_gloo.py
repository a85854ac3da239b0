"""N > 1 bookkeeping on CPU: two gloo ranks shard the query stream, answer their shards (with the
oracle standing in for the device), and reduce times / checksums exactly like bench.py does."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2109_14807_b200.shard import shard_range


def test_shard_ranges_tile_the_stream():
    for n in (0, 1, 7, 10**9 + 3):
        for w in (1, 2, 3, 4, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out_dir):
    import torch.distributed as dist
    import oracle
    import synth
    from paper_2109_14807_b200.shard import reduce_times_and_checksum, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS[2].scaled(N=128)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    f = synth.build_factors(cfg, nxy, bins)
    i0, i1 = shard_range(n, rank, world)
    recs = synth.gen_queries(cfg, bins, i0, i1)  # counter-based: independent of the split
    res = oracle.query_batch(oracle.desc_of(cfg), f.C, f.X, f.Y, f.Z, recs)
    np.save(os.path.join(out_dir, f"res_{rank}.npy"), res)
    (tmax,), total = reduce_times_and_checksum([float(rank + 1)], float(res.sum()))
    if rank == 0:
        np.save(os.path.join(out_dir, "reduced.npy"), np.array([tmax, total]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_gloo_ranks_match_one_process(tmp_path):
    import oracle
    import synth
    n = 20_011
    mp.spawn(_worker, args=(2, _free_port(), n, str(tmp_path)), nprocs=2, join=True)
    parts = [np.load(tmp_path / f"res_{r}.npy") for r in range(2)]
    cfg = synth.CONFIGS[2].scaled(N=128)
    nxy = synth.make_map(cfg)
    bins = synth.bin_map(cfg, nxy)
    f = synth.build_factors(cfg, nxy, bins)
    full = oracle.query_batch(oracle.desc_of(cfg), f.C, f.X, f.Y, f.Z, synth.gen_queries(cfg, bins, 0, n))
    assert np.concatenate(parts).tobytes() == full.tobytes()  # per-query results independent of the split
    tmax, total = np.load(tmp_path / "reduced.npy")
    assert tmax == 2.0                                         # MAX over ranks of the step time
    assert total == pytest.approx(parts[0].sum() + parts[1].sum(), rel=1e-15)


def test_spatial_owner_partitions_the_stream():
    """Spatial sharding: every query has exactly one owner (a function of its centre), strips are
    balanced for the configs' uniformly placed centres, world 1 owns everything."""
    import synth
    from paper_2109_14807_b200.shard import spatial_owner
    cfg = synth.CONFIGS[5]
    recs = synth.gen_queries(cfg, None, 0, 400_000)
    for w in (1, 2, 4, 8):
        own = spatial_owner(recs["u"], cfg.N, w)
        assert own.min() >= 0 and own.max() <= w - 1
        counts = np.bincount(own, minlength=w)
        assert counts.sum() == recs.shape[0]
        assert np.abs(counts / recs.shape[0] - 1.0 / w).max() < 0.01
    assert (spatial_owner(recs["u"], cfg.N, 1) == 0).all()
    # strips: owner is monotone in u and wraps
    u = np.array([0.0, 511.99, 512.0, 4095.99, 4096.0, -1.0])
    assert spatial_owner(u, 4096, 8).tolist() == [0, 0, 1, 7, 0, 7]


def test_bench_spatial_shards_cover_the_stream_exactly():
    """bench.py's spatial shards of a W-rank job: disjoint, in stream order, and together exactly the
    stream (every query answered once), for W = 2 and 3."""
    import sys
    import os
    import synth
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    cfg = synth.CONFIGS[2]
    n = 50_000
    bins = synth.bin_map(cfg, synth.make_map(cfg))
    full = synth.gen_queries(cfg, bins, 0, n)
    for w in (2, 3):
        parts = [bench.spatial_shard(cfg, bins, n, r, w).numpy().view(synth.QREC).reshape(-1) for r in range(w)]
        assert sum(p.shape[0] for p in parts) == n
        merged = np.concatenate(parts)
        key = lambda a: np.sort(a.view(np.dtype((np.void, 16))))  # noqa: E731
        assert np.array_equal(key(merged), key(full))
        for r, p in enumerate(parts):  # stream order kept inside a shard, and every record in its strip
            pos = np.flatnonzero(np.isin(full.view(np.dtype((np.void, 16))), p.view(np.dtype((np.void, 16)))))
            assert np.all(np.diff(pos) > 0)
            assert (np.minimum((p["u"] * w / cfg.N).astype(int), w - 1) == r).all()
