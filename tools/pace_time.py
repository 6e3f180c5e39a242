"""Device time of oz_gemm steps at n = 8192 for the headline and the FP64-level
configuration under the current OZ_PACE_SLACK (read at import).  usage: pace_time.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs, _time_steps  # noqa: E402

n = 8192
A, B = gpu_inputs(torch, n, n, n, 0.5, 1, "cuda")
f8, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp32")
for name, cfg, steps in (("fixed11", oz.GemmConfig(f8, f32, pair_cutoff=11, slice_exponents="fixed"), 12),
                         ("defaults", oz.GemmConfig(f8, f32), 4),
                         ("fixed11", oz.GemmConfig(f8, f32, pair_cutoff=11, slice_exponents="fixed"), 12)):
    _time_steps(torch, oz, A, B, cfg, 2)
    ms, st = _time_steps(torch, oz, A, B, cfg, steps)
    print(f"slack={os.environ.get('OZ_PACE_SLACK', '2')} {name}: {ms:.2f} ms/step "
          f"({2 * n ** 3 / ms / 1e9:.2f} TF/s, K3 {st.t_gemm * 1e3:.2f} ms)", flush=True)
