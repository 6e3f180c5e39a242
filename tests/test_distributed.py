"""2-D output-tile sharding (row (e) of SURVEY.md §8) on CPU with the gloo
backend: each rank receives its A row-panel / B column-panel through the same
TileGrid.distribute_panels the NCCL path uses, computes its C tile (here with
the CPU oracle, standing in for the per-GPU kernels), and the assembled C is
bitwise equal to the single-process result — no reduction anywhere."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_00441_b200.distributed import TileGrid, split_extent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_grid_shapes():
    assert (TileGrid.for_world(1).rows, TileGrid.for_world(1).cols) == (1, 1)
    assert (TileGrid.for_world(2).rows, TileGrid.for_world(2).cols) == (1, 2)
    assert (TileGrid.for_world(4).rows, TileGrid.for_world(4).cols) == (2, 2)
    assert (TileGrid.for_world(8).rows, TileGrid.for_world(8).cols) == (2, 4)
    g = TileGrid(2, 4)
    assert [g.coords(r) for r in range(8)] == [(i, j) for i in range(2) for j in range(4)]
    assert g.row_members(1) == [4, 5, 6, 7] and g.col_members(2) == [2, 6]


@pytest.mark.parametrize("total,parts", [(1000, 3), (8192, 4), (128, 2), (300, 8)])
def test_split_extent_covers_exactly(total, parts):
    spans = [split_extent(total, parts, i) for i in range(parts)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    # 128-aligned boundaries (C tiles align with the MMA tiles)
    assert all(lo % 128 == 0 for lo, _ in spans if lo < total)


def _worker(rank, world, port, m, n, k, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle

    grid = TileGrid.for_world(world)
    groups = grid.make_groups(dist)
    (r0, r1), (c0, c1) = grid.tile_extent(rank, m, n)
    rng = np.random.default_rng(7)
    A = (rng.random((m, k)) - 0.5) * np.exp(1.0 * rng.standard_normal((m, k)))
    B = (rng.random((k, n)) - 0.5) * np.exp(1.0 * rng.standard_normal((k, n)))
    # only the panel roots hold real data; everyone else receives it by broadcast
    Ap = torch.from_numpy(np.ascontiguousarray(A[r0:r1])) if grid.is_row_root(rank) else torch.empty(r1 - r0, k,
                                                                                                    dtype=torch.float64)
    Bp = torch.from_numpy(np.ascontiguousarray(B[:, c0:c1])) if grid.is_col_root(rank) else torch.empty(k, c1 - c0,
                                                                                                      dtype=torch.float64)
    grid.distribute_panels(dist, groups, rank, Ap, Bp)
    assert np.array_equal(Ap.numpy(), A[r0:r1]) and np.array_equal(Bp.numpy(), B[:, c0:c1])
    C, info = oracle.oz_gemm(Ap.numpy(), Bp.numpy(), nthreads=1)
    np.save(os.path.join(out_dir, f"tile{rank}.npy"), C)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tile_sharded_equals_single_process(tmp_path, world):
    m, n, k = 300, 260, 96
    mp.spawn(_worker, args=(world, _free_port(), m, n, k, str(tmp_path)), nprocs=world, join=True)
    import oracle

    rng = np.random.default_rng(7)
    A = (rng.random((m, k)) - 0.5) * np.exp(1.0 * rng.standard_normal((m, k)))
    B = (rng.random((k, n)) - 0.5) * np.exp(1.0 * rng.standard_normal((k, n)))
    Cfull, _ = oracle.oz_gemm(A, B)
    grid = TileGrid.for_world(world)
    C = np.empty((m, n))
    for r in range(world):
        (r0, r1), (c0, c1) = grid.tile_extent(r, m, n)
        C[r0:r1, c0:c1] = np.load(tmp_path / f"tile{r}.npy")
    # The per-tile slicing differs from the full-matrix slicing only in the global s
    # (zero-padded pairs), which is result-neutral: the tiles must match bitwise.
    assert np.array_equal(C.view(np.uint64), Cfull.view(np.uint64))
