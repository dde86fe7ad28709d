"""View-sharded multi-GPU uplift: host-side plumbing around the C ABI.

Views are independent -- e_i(v,p) depends on one view and all Gaussians (Eq. 2,
P:68-72) -- so rank r of P takes the views v = r (mod P) and accumulates a full fp32 W/Z
partial over them (Eq. 5 / Algorithm 1 lines 5-12).  Eq. 5 is a sum over views,
so the partials add: one reduce-scatter per buffer hands rank r the rows
[r*Npad/P, (r+1)*Npad/P) of the total, on which it runs Eq. 6 locally.  With
the NCCL backend the collective runs over NVLink/NVSwitch; the same functions run on gloo
(CPU) in the tests.

Only index arithmetic and collectives live here; every step of the method runs in the CUDA
library (`uplift.SparseUplift`).
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple


def views_for_rank(num_views: int, rank: int, world: int) -> List[int]:
    """Interleaved view shard v = rank (mod world): orbit cameras alternate around the scene,
    so neighbouring (similar-cost) views land on different ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, num_views, world))


def padded_rows(num_gaussians: int, world: int) -> int:
    """Accumulator rows: the smallest multiple of `world` >= num_gaussians (>= world)."""
    return max(1, int(math.ceil(num_gaussians / world))) * world


def row_shard(num_gaussians: int, rank: int, world: int) -> Tuple[int, int]:
    """(first_row, num_rows) of rank's Gaussian shard after the reduce-scatter."""
    n = padded_rows(num_gaussians, world) // world
    return rank * n, n


def reduce_scatter_accumulators(W, Z, W_shard, Z_shard, group=None) -> None:
    """Sum the ranks' W [Npad, L] and Z [Npad] partials; rank r receives rows of its shard.
    Two calls (not one packed buffer) keep W's rows 256-B aligned."""
    import torch.distributed as dist
    dist.reduce_scatter_tensor(W_shard, W, op=dist.ReduceOp.SUM, group=group)
    dist.reduce_scatter_tensor(Z_shard, Z, op=dist.ReduceOp.SUM, group=group)


def all_gather_codes(atoms_shard, coefs_shard, atoms_all, coefs_all, group=None) -> None:
    """Optional: every rank gets every Gaussian's K-sparse code ([Npad, K] each)."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(atoms_all, atoms_shard, group=group)
    dist.all_gather_into_tensor(coefs_all, coefs_shard, group=group)


def exchange_accumulators(W, rank: int, world: int, device: int, group=None, abi_mod=None):
    """Share every rank's accumulator with every other rank through CUDA IPC (NVLink / NVSwitch
    peer mappings): export the local W's allocation handle, all-gather (handle, offset) over the
    process group, open the peers' handles.  Returns (pointers in rank order, mapping bases to
    close); pointer `rank` is the local one."""
    import torch.distributed as dist
    if abi_mod is None:
        from . import abi as abi_mod
    local = W.data_ptr()
    try:
        mine = abi_mod.scoup_ipc_export(local)
    except Exception:  # still join the collective, so that no rank waits for this one
        mine = None
    every = [None] * world
    dist.all_gather_object(every, mine, group=group)
    if any(x is None for x in every):
        raise RuntimeError("a rank could not export its accumulator for CUDA IPC")
    ptrs, bases = [], []
    for q, (handle, off) in enumerate(every):
        if q == rank:
            ptrs.append(local)
            continue
        p, b = abi_mod.scoup_ipc_import(device, handle, off)
        ptrs.append(p)
        bases.append(b)
    return ptrs, bases


def fused_reduce_finalize(up, peers, first_row: int, num_rows: int, level: int = 0, out_atoms=None,
                          out_coefs=None, group=None):
    """SURVEY.md §8(e)'s fused exchange: after a barrier (every rank's partial is complete), one
    kernel reads this rank's rows from all P partials over the peer mappings, sums them in rank
    order and runs Eq. 6 -- no reduced shard is written; a second barrier keeps the peers' W
    alive until every rank has read it."""
    import torch
    import torch.distributed as dist
    from . import abi
    if out_atoms is None:
        out_atoms = torch.empty((num_rows, up.K), dtype=torch.int32, device=up.device)
    if out_coefs is None:
        out_coefs = torch.empty((num_rows, up.K), dtype=torch.float32, device=up.device)
    up.stream.synchronize()
    dist.barrier(group=group)
    abi.scoup_uplift_finalize_topk_peers(up._h, level, first_row, num_rows, peers, out_atoms, out_coefs)
    dist.barrier(group=group)
    return out_atoms, out_coefs


class ShardedUplift:
    """One rank of a view-sharded uplift of one semantic level.

        up = ShardedUplift(gaussians, L, K, rank, world, device=local_rank)
        up.add_views(cams_of_my_views, region_ids, codes)    # views_for_rank(...)
        atoms, coefs = up.finalize()                         # rows row_shard(G, rank, world)
    """

    def __init__(self, gaussians, L: int, K: int, rank: int, world: int, device: int = 0,
                 group=None, stream=None):
        import torch
        from .uplift import SparseUplift
        self.rank, self.world, self.group = rank, world, group
        self.G = int(gaussians.means.shape[0])
        self.Npad = padded_rows(self.G, world)
        self.first_row, self.num_rows = row_shard(self.G, rank, world)
        self.up = SparseUplift(gaussians, L, K, device=device, rows_padded=self.Npad, stream=stream)
        dev = self.up.device
        if world > 1:
            self.W_shard = torch.empty((self.num_rows, L), dtype=torch.float32, device=dev)
            self.Z_shard = torch.empty((self.num_rows,), dtype=torch.float32, device=dev)

    def add_views(self, cameras: Sequence, region_ids, codes, contributions_out=None):
        self.up.add_views(cameras, region_ids, codes, contributions_out)

    def reset(self):
        self.up.reset()

    def finalize(self, out_atoms=None, out_coefs=None):
        """Reduce-scatter the partials (world > 1) and run Eq. 6 on this rank's rows."""
        if self.world == 1:
            return self.up.finalize(0, self.G, out_atoms=out_atoms, out_coefs=out_coefs)
        reduce_scatter_accumulators(self.up.W, self.up.Z, self.W_shard, self.Z_shard, self.group)
        return self.up.finalize(self.first_row, self.num_rows, W_rows=self.W_shard, Z_rows=self.Z_shard,
                                out_atoms=out_atoms, out_coefs=out_coefs)

    def stats(self) -> dict:
        return self.up.stats()

    def close(self):
        self.up.close()
