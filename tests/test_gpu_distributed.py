"""Multi-rank 2-D C-tile sharding through the real GPU kernels on ONE B200
(every rank on cuda:0, gloo carrying the CUDA panels): the tiles assembled
from the ranks are bitwise the single-GPU C, and bench.py's config-5
strong-scaling mode runs end to end under torchrun with a bitwise parity
sample (BASELINE.json configs[4]; the 8-GPU NCCL run uses the same code)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import spread_matrix

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(m, n, k):
    rng = np.random.default_rng(11)
    return spread_matrix(rng, m, k, 1.0), spread_matrix(rng, k, n, 1.0)


def _worker(rank, world, port, m, n, k, cfg_kw, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2508_00441_b200 as oz
    from paper_2508_00441_b200.distributed import TileGrid, oz_gemm_tile

    grid = TileGrid.for_world(world)
    groups = grid.make_groups(dist)
    (r0, r1), (c0, c1) = grid.tile_extent(rank, m, n)
    A, B = _inputs(m, n, k)
    Ap = torch.empty((r1 - r0, k), dtype=torch.float64, device="cuda")
    Bp = torch.empty((k, c1 - c0), dtype=torch.float64, device="cuda")
    if grid.is_row_root(rank):
        Ap.copy_(torch.from_numpy(np.ascontiguousarray(A[r0:r1])))
    if grid.is_col_root(rank):
        Bp.copy_(torch.from_numpy(np.ascontiguousarray(B[:, c0:c1])))
    grid.distribute_panels(dist, groups, rank, Ap, Bp)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), **cfg_kw)
    C, _ = oz_gemm_tile(Ap, Bp, cfg)
    np.save(os.path.join(out_dir, f"tile{rank}.npy"), C.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cfg_kw", [{}, {"pair_cutoff": 9, "slice_exponents": "fixed"}, {"k_block": 256}],
                         ids=["defaults", "fixed9", "kb256"])
def test_tiles_on_gpu_equal_single_gpu(cuda, tmp_path, world, cfg_kw):
    import paper_2508_00441_b200 as oz
    from paper_2508_00441_b200.distributed import TileGrid

    m, n, k = 700, 600, 900
    mp.spawn(_worker, args=(world, _free_port(), m, n, k, cfg_kw, str(tmp_path)), nprocs=world, join=True)
    A, B = _inputs(m, n, k)
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), **cfg_kw)
    Cfull = oz.oz_gemm(A, B, cfg).C
    grid = TileGrid.for_world(world)
    C = np.full((m, n), np.nan)
    for r in range(world):
        (r0, r1), (c0, c1) = grid.tile_extent(r, m, n)
        C[r0:r1, c0:c1] = np.load(tmp_path / f"tile{r}.npy")
    assert np.array_equal(C.view(np.uint64), Cfull.view(np.uint64))


@pytest.mark.parametrize("extra", [[], ["--pair-cutoff", "10", "--slice-exponents", "fixed"]],
                         ids=["defaults", "fixed10"])
def test_bench_strong_two_ranks(cuda, extra):
    """bench.py config-5 mode under torchrun (2 ranks on cuda:0): one JSON line,
    strong scaling over a 1 x 2 tile grid, bitwise parity sample, e2e keys."""
    env = dict(os.environ, OZ_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--size", "2048", "--steps", "2", "--warmup", "1", "--no-variants", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["tile"] == [2048, 1024]
    assert d["parity"]["bitwise_equal"] is True and d["parity"]["mismatches"] == 0
    assert d["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 8 * 2048 * 2048
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 8 * 2048 * 2048  # A at the row root, B halves at the column roots
