"""Per-pass device times (split phase, pair GEMM) of one panelled oz_gemm_device
call, plus host wall-clock around the enqueue loop.  usage: pass_times.py n [cutoff]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import ozgemm  # noqa: E402
from bench import fill_cols, fill_rows  # noqa: E402

n = int(sys.argv[1])
cut = int(sys.argv[2]) if len(sys.argv) > 2 else None
A = torch.empty((n, n), dtype=torch.float64, device="cuda")
B = torch.empty((n, n), dtype=torch.float64, device="cuda")
fill_rows(torch, A, 0, n, 0.5, 1000, "cuda")
fill_cols(torch, B, 0, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=cut)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = ozgemm._enqueue(torch, A, B, cfg, C, True, None, True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: host enqueue {t1 - t0:.3f} s, total {t2 - t0:.3f} s, mp={st['mp']} np={st['np']}")
    for i, e in enumerate(st["evs"]):
        print(f"  pass {i:2d} split {e[0].elapsed_time(e[1]):9.2f} ms  gemm {e[1].elapsed_time(e[2]):9.2f} ms")
