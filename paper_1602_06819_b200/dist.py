"""Multi-GPU online insert for partitioned graphs (Alg. 3 + Alg. 5 across ranks).

One process per GPU (torchrun), every rank holding a full replica of the graph and making the same
calls with the same inputs.  Partitioned graphs shard the P partition searches (below);
unpartitioned graphs shard the queries of the batch instead (same stages, cand gathered by query).  A batch is inserted in the three C-ABI stages of include/knng.h with
two all-gathers in between (torch.distributed, NCCL over NVLink on a GPU box):

  1. graph_insert_stage_search  -- this rank's partitions [r P/G, (r+1) P/G)      -> cand [B][P/G][k]
  2. all-gather cand                                                          -> [G][B][P/G][k]
  3. graph_insert_stage_update  -- merge (identical everywhere), new rows + balls of the query shard
  4. all-gather new rows and proposals (S = ceil(B/G) slots per rank)    -> [G*S][k], [G*S][ballmax]
  5. graph_insert_stage_commit  -- write the new rows, apply all proposals, place the points

The exchange carries B*P*k*8 + G*S*ballmax*8 bytes per batch (C3: 5.2 MB + 7.2 MB), the only
data-path collectives of the path.  Results are identical for every G (tested by emulating G ranks
on one GPU, and the decomposition itself on CPU with gloo + the oracle).
"""
from __future__ import annotations

import torch


def owned_partitions(P, world, rank):
    """Partitions [lo, hi) searched by `rank` (P must be a multiple of the world size)."""
    if P % world:
        raise ValueError("P=%d is not a multiple of the world size %d" % (P, world))
    per = P // world
    return rank * per, (rank + 1) * per


def query_shard(B, world, rank):
    """Queries [lo, hi) whose update balls `rank` runs, and the equal per-rank slot count S."""
    S = -(-B // world) if B else 0
    lo = min(rank * S, B)
    return lo, min(lo + S, B), S


class TorchComm:
    """All-gather along dim 0 over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather(self, t):
        t = t.contiguous()
        if t.is_cuda and self.dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return out
        # gloo (CPU tests / plumbing tests): host-staged
        h = t.cpu()
        parts = [torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(parts, h, group=self.group)
        return torch.cat(parts, 0).to(t.device)


def _i32(n_elems_shape, device):
    return torch.empty(n_elems_shape, dtype=torch.int32, device=device)


def _sync():
    """Buffers made by torch (its stream) are consumed by the library (its own stream)."""
    if torch.cuda.is_available():
        torch.cuda.current_stream().synchronize()


def library_graph(points, k, device, capacity=0, stream=None, group=None, metric=None):
    """This rank's replica with the LIBRARY-owned NCCL communicator: rank 0 makes the 128-byte NCCL id
    (graph_nccl_unique_id), torch.distributed broadcasts it, and every rank's graph_init joins the
    communicator.  graph_insert_batch on the returned handle is then the whole distributed insert in
    one C-ABI call (all-gathers on the handle's stream, no host sync between the stages)."""
    import torch.distributed as dist
    from .knng import KnngGraph, nccl_unique_id
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    idt = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        idt[:] = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        idd = idt.cuda()
        dist.broadcast(idd, 0, group=group)
        idt = idd.cpu()
    else:
        dist.broadcast(idt, 0, group=group)
    return KnngGraph(points, k, device=device, capacity=capacity, stream=stream, rank=rank, world=world, metric=metric,
                     nccl_id=bytes(idt.numpy().tobytes()))


class DistributedGraph:
    """A rank's replica of a graph driven by the STAGED C-ABI calls and torch.distributed all-gathers
    (the host-orchestrated form of the library's distributed insert: plumbing tests, gloo)."""

    def __init__(self, graph, comm):
        self.g = graph
        self.comm = comm

    def insert_batch(self, points, speedup, e_num, e_den, depth, seed):
        _, med = self.g.partition()
        return insert_batch_staged([self.g], [self.comm.rank], self.comm.world, points, speedup, e_num, e_den,
                                   depth, seed, 0 if med is None else len(med), allgather=self.comm.allgather)


def insert_batch_staged(graphs, ranks, world, points, speedup, e_num, e_den, depth, seed, P, allgather=None):
    """Run the three stages for the replicas `graphs` (one per entry of `ranks`) of a `world`-rank job.

    Partitioned graphs (P > 0) shard the partitions (Alg. 3); unpartitioned graphs shard the
    queries of the batch (every replica holds the whole graph; the batch is one snapshot batch).
    With one replica per process, `allgather` is the communicator's all-gather.  With every rank's
    replica in this process (emulation on one GPU: len(graphs) == world), the gathers are the
    concatenation of the ranks' buffers in rank order -- the same layout an all-gather produces;
    nothing waits on another launch.
    Returns the per-replica stage stats.
    """
    B = len(points)
    k = graphs[0].k
    dev = "cuda"
    ballmax = graphs[0].ball_bound(depth)
    S = query_shard(B, world, 0)[2]
    stats = [dict() for _ in graphs]

    def gather(bufs):
        if allgather is not None:
            return allgather(bufs[0])
        return torch.cat(bufs, 0)

    # 1-2: searches (partition-sharded, or query-sharded), all-gather of the candidates
    cis, cks = [], []
    for g, r in zip(graphs, ranks):
        if P > 0:
            lo, hi = owned_partitions(P, world, r)
            cis.append(torch.full((B, hi - lo, k), -1, dtype=torch.int32, device=dev))
            cks.append(torch.zeros((B, hi - lo, k), dtype=torch.int32, device=dev))
        else:
            cis.append(torch.full((S, 1, k), -1, dtype=torch.int32, device=dev))
            cks.append(torch.zeros((S, 1, k), dtype=torch.int32, device=dev))
    _sync()
    for i, (g, r) in enumerate(zip(graphs, ranks)):
        if P > 0:
            lo, hi = owned_partitions(P, world, r)
            stats[i]["search"] = g.stage_search(points, speedup, e_num, e_den, depth, seed, lo, hi, cis[i], cks[i])
        else:
            qlo, qhi, _ = query_shard(B, world, r)
            stats[i]["search"] = g.stage_search(points, speedup, e_num, e_den, depth, seed, 0, 1, cis[i], cks[i],
                                                qlo, qhi)
    ci_all, ck_all = gather(cis), gather(cks)      # P > 0: [G][B][P/G][k]; else [G*S][1][k] (row b = query b)
    # 3-4: merge + new rows + balls of the query shard, all-gather of the proposals
    bufs = [(torch.zeros((S, ballmax, 2), dtype=torch.int32, device=dev),
             torch.zeros((S,), dtype=torch.int32, device=dev),
             torch.full((S, k), -1, dtype=torch.int32, device=dev),
             torch.zeros((S, k), dtype=torch.int32, device=dev)) for _ in graphs]
    _sync()
    for i, (g, r) in enumerate(zip(graphs, ranks)):
        qlo, qhi, _ = query_shard(B, world, r)
        props, cnt, nid, nkey = bufs[i]
        stats[i]["update"] = g.stage_update(speedup, e_num, e_den, depth, seed, world if P > 0 else 1, ci_all, ck_all,
                                            qlo, qhi, props, cnt, nid, nkey)
    props_all = gather([b[0] for b in bufs])
    cnt_all = gather([b[1] for b in bufs])
    nid_all = gather([b[2] for b in bufs])
    nkey_all = gather([b[3] for b in bufs])
    _sync()
    # 5: commit everywhere
    for i, g in enumerate(graphs):
        stats[i]["commit"] = g.stage_commit(speedup, e_num, e_den, depth, seed, props_all.shape[0], props_all, cnt_all,
                                            nid_all, nkey_all)
    return stats
