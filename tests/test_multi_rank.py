"""N > 1 path on the CPU: world_size-2 (and 3) gloo process groups run the same host-side
sharding + collective code bench.py uses (paper_2605_13600_b200/distributed.py) on oracle
partials.  The GPU kernels are not involved (no GPU here); what is checked is that view
sharding covers every view once, that the reduce-scatter of per-rank partials equals the
single-process accumulation (Eq. 5 is a sum over views), and that each rank's
shard Top-K plus the codes all-gather reproduce the single-process codes (Eq. 6)."""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2605_13600_b200 import distributed as D  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_view_and_row_sharding_cover_everything():
    for V in [0, 1, 4, 5, 300]:
        for P in [1, 2, 3, 8]:
            got = sorted(v for r in range(P) for v in D.views_for_rank(V, r, P))
            assert got == list(range(V))
            sizes = [len(D.views_for_rank(V, r, P)) for r in range(P)]
            assert max(sizes) - min(sizes) <= 1
    for G in [1, 7, 2000, 3_000_001]:
        for P in [1, 2, 3, 8]:
            Npad = D.padded_rows(G, P)
            assert Npad % P == 0 and Npad >= G and Npad - G < P
            rows = [D.row_shard(G, r, P) for r in range(P)]
            assert rows[0][0] == 0 and all(a + n == b for (a, n), (b, _) in zip(rows, rows[1:]))
            assert rows[-1][0] + rows[-1][1] == Npad
    with pytest.raises(ValueError):
        D.views_for_rank(4, 2, 2)


def _worker(rank, world, port, result_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    from paper_2605_13600_b200 import synth
    from helpers import compare_codes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS["tiny"].with_(num_views=5, unassigned_frac=0.1)
        scene = synth.make_scene(cfg, 0)
        g = scene.gaussians
        G, L, K = g.count, cfg.L, cfg.K
        mine = D.views_for_rank(cfg.num_views, rank, world)
        maps = synth.make_region_maps_numpy(cfg, seed=0, views=mine)
        codes = synth.make_codes(cfg, seed=0, views=mine)
        Npad = D.padded_rows(G, world)
        first, n = D.row_shard(G, rank, world)
        W = torch.zeros((Npad, L), dtype=torch.float64)
        Z = torch.zeros((Npad,), dtype=torch.float64)
        if mine:
            Wp, Zp, frags = oracle.uplift_accumulate(g, [scene.cameras[v] for v in mine], maps, codes.atoms,
                                                     codes.coefs, codes.row0, codes.num_regions, L, K)
            W[:G] = torch.from_numpy(Wp)
            Z[:G] = torch.from_numpy(Zp)
        Ws = torch.empty((n, L), dtype=torch.float64)
        Zs = torch.empty((n,), dtype=torch.float64)
        D.reduce_scatter_accumulators(W, Z, Ws, Zs)
        # single-process reference (every view on every rank)
        maps_all = synth.make_region_maps_numpy(cfg, seed=0)
        codes_all = synth.make_codes(cfg, seed=0)
        Wf, Zf, _ = oracle.uplift_accumulate(g, scene.cameras, maps_all, codes_all.atoms, codes_all.coefs,
                                             codes_all.row0, codes_all.num_regions, L, K)
        valid = max(0, min(n, G - first))
        assert np.allclose(Ws[:valid].numpy(), Wf[first:first + valid], rtol=1e-12, atol=1e-15)
        assert np.allclose(Zs[:valid].numpy(), Zf[first:first + valid], rtol=1e-12, atol=1e-15)
        assert torch.all(Ws[valid:] == 0) and torch.all(Zs[valid:] == 0)
        # shard Top-K (Eq. 6) then all-gather of the codes
        a_s, c_s = oracle.topk(Ws.numpy(), K)
        atoms_all = torch.empty((Npad, K), dtype=torch.int64)
        coefs_all = torch.empty((Npad, K), dtype=torch.float64)
        D.all_gather_codes(torch.from_numpy(a_s.astype(np.int64)), torch.from_numpy(c_s), atoms_all, coefs_all)
        bad, ties, worst = compare_codes(atoms_all[:G].numpy(), coefs_all[:G].numpy(), Wf, K)
        assert bad == 0, worst
        with open(os.path.join(result_dir, f"ok{rank}"), "w") as fh:
            fh.write(f"{len(mine)} views, rows {first}+{n}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_view_sharded_reduce_scatter_matches_single_process(world, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert sorted(os.listdir(tmp_path)) == [f"ok{r}" for r in range(world)]


class _FakeW:
    def __init__(self, p):
        self._p = p

    def data_ptr(self):
        return self._p


class _FakeAbi:
    """Stands in for the CUDA IPC calls: rank q's handle encodes q; importing it 'maps' it at
    0x1000 * (q + 1) + offset."""

    def __init__(self, rank):
        self.rank = rank
        self.opened = []

    def scoup_ipc_export(self, dptr):
        return bytes([self.rank]) * 64, 16 * (self.rank + 1)

    def scoup_ipc_import(self, device, handle, offset):
        q = handle[0]
        assert handle == bytes([q]) * 64 and q != self.rank and offset == 16 * (q + 1)
        self.opened.append(q)
        return 0x1000 * (q + 1) + offset, 0x1000 * (q + 1)


def _exchange_worker(rank, world, port, result_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = _FakeAbi(rank)
        ptrs, bases = D.exchange_accumulators(_FakeW(0xABC0 + rank), rank, world, device=0, abi_mod=fake)
        expect = [0xABC0 + q if q == rank else 0x1000 * (q + 1) + 16 * (q + 1) for q in range(world)]
        ok = ptrs == expect and sorted(fake.opened) == [q for q in range(world) if q != rank] and \
            bases == [0x1000 * (q + 1) for q in range(world) if q != rank]
        with open(os.path.join(result_dir, f"ex{rank}.txt"), "w") as fh:
            fh.write("ok" if ok else f"bad {ptrs} {bases}")
    finally:
        dist.destroy_process_group()


class _FailingAbi(_FakeAbi):
    def scoup_ipc_export(self, dptr):
        if self.rank == 1:
            raise RuntimeError("no IPC here")
        return super().scoup_ipc_export(dptr)


def _exchange_fail_worker(rank, world, port, result_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            D.exchange_accumulators(_FakeW(1), rank, world, device=0, abi_mod=_FailingAbi(rank))
            msg = "no error"
        except RuntimeError as ex:
            msg = "raised" if "export" in str(ex) or "IPC" in str(ex) else str(ex)
        with open(os.path.join(result_dir, f"fx{rank}.txt"), "w") as fh:
            fh.write(msg)
    finally:
        dist.destroy_process_group()


def test_accumulator_exchange_failure_is_collective(tmp_path):
    """If one rank cannot export its accumulator, every rank raises (none is left waiting in a
    collective), so the caller can fall back to the NCCL reduce-scatter on all ranks."""
    mp.spawn(_exchange_fail_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    for r in range(3):
        assert open(os.path.join(tmp_path, f"fx{r}.txt")).read() == "raised"


@pytest.mark.parametrize("world", [2, 3])
def test_accumulator_exchange_over_gloo(tmp_path, world):
    """The host side of the fused cross-rank reduction (distributed.exchange_accumulators): every
    rank ends with one pointer per rank in rank order -- its own W and the peers' IPC mappings --
    and opens exactly the other ranks' handles (CUDA IPC calls replaced by a recording fake)."""
    mp.spawn(_exchange_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert open(os.path.join(tmp_path, f"ex{r}.txt")).read() == "ok"
