"""The multi-GPU decomposition on CPU: world_size-2 gloo processes run the staged batch
(partition-sharded searches, all-gathered candidates, query-sharded update balls, all-gathered
proposals, commit) with the oracle as the per-rank compute and the product's exchange helpers
(paper_1602_06819_b200.dist); every rank must end with the monolithic oracle's graph."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen as D
from oracle import oracle as O
from paper_1602_06819_b200.dist import TorchComm, owned_partitions, query_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(cfg_name):
    cfg = D.CONFIGS[cfg_name].with_sizes(n0=1200 if cfg_name == "C3" else 700, n_insert=140)
    X = D.initial_points(cfg)
    S = D.stream_points(cfg, 0, cfg.n_insert)
    o = O.OracleGraph(cfg.metric, X, cfg.k, capacity=cfg.n0 + cfg.n_insert + 4)
    o.init_exact(1)
    part, med, _ = o.partition_kmedoids(cfg.P, cfg.imbalance, 2, cfg.part_seed)
    o.set_partition(part, med)
    return cfg, S, o


def _worker(rank, world, port, cfg_name, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorchComm()
    cfg, S, o = _setup(cfg_name)
    for lo, hi in ((0, 61), (61, 62), (62, 140)):
        pts = S[lo:hi]
        B = hi - lo
        ballmax = o.ball_bound(cfg.depth)
        plo, phi = owned_partitions(cfg.P, world, rank)
        ci, ck = o.stage_search(pts, plo, phi, cfg.speedup, cfg.e_num, cfg.e_den, cfg.search_seed)
        ci_all = comm.allgather(torch.from_numpy(ci)).numpy()
        ck_all = comm.allgather(torch.from_numpy(ck.view(np.int32))).numpy().view(np.uint32)
        C_i, C_k = O.merge_candidates(cfg.metric, ci_all, ck_all, world, cfg.P, cfg.k)
        qlo, qhi, Sq = query_shard(B, world, rank)
        props, cnt = o.stage_update(C_i, C_k, qlo, qhi, cfg.depth, ballmax)
        pp = np.zeros((Sq, ballmax, 2), np.int32)
        cc = np.zeros(Sq, np.int32)
        pp[:len(props)] = props
        cc[:len(cnt)] = cnt
        pa = comm.allgather(torch.from_numpy(pp)).numpy()
        ca = comm.allgather(torch.from_numpy(cc)).numpy()
        o.stage_commit(pa, ca, ballmax)
    np.save(os.path.join(out_dir, "ids_%d.npy" % rank), o.ids[:o.n])
    np.save(os.path.join(out_dir, "keys_%d.npy" % rank), o.keys[:o.n])
    np.save(os.path.join(out_dir, "part_%d.npy" % rank), o.part_of[:o.n])
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["C3", "C4"])
def test_two_rank_decomposition_equals_single_process(cfg_name, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), cfg_name, str(tmp_path)), nprocs=world, join=True)
    cfg, S, o = _setup(cfg_name)
    for lo, hi in ((0, 61), (61, 62), (62, 140)):
        o.insert_batch(S[lo:hi], cfg.speedup, cfg.e_num, cfg.e_den, cfg.depth, cfg.search_seed, 2)
    for r in range(world):
        assert (np.load(tmp_path / ("ids_%d.npy" % r)) == o.ids[:o.n]).all()
        assert (np.load(tmp_path / ("keys_%d.npy" % r)) == o.keys[:o.n]).all()
        assert (np.load(tmp_path / ("part_%d.npy" % r)) == o.part_of[:o.n]).all()


def test_shard_helpers():
    assert [owned_partitions(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    with pytest.raises(ValueError):
        owned_partitions(8, 3, 0)
    for B in (0, 1, 7, 8, 1024, 8192, 8193):
        for world in (1, 2, 4, 8):
            sh = [query_shard(B, world, r) for r in range(world)]
            covered = [q for lo, hi, _ in sh for q in range(lo, hi)]
            assert covered == list(range(B))
            assert all(hi - lo <= s for lo, hi, s in sh)
