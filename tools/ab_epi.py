"""A/B: epilogue warps of the N = 192 CTA-pair kernel (oz_set_epilogue_warps),
n = 8192, reference defaults and pair_cutoff = 11; alternating runs, device
time of the pair GEMM per call, C compared bitwise between the variants."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from bench import gpu_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
for cut in (None, 11):
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), pair_cutoff=cut)
    ref = {}
    for rep in range(3):
        for w in (8, 12):
            _lib.call("oz_set_epilogue_warps", w)
            oz.oz_gemm_device(A, B, cfg, out=C)
            ts = []
            for _ in range(3):
                _, st = oz.oz_gemm_device(A, B, cfg, out=C)
                ts.append(st.t_gemm * 1e3)
            if w not in ref:
                ref[w] = C.clone()
            print(f"cut={cut} epi={w}: K3 {min(ts):8.2f} ms (runs {[round(t, 2) for t in ts]})", flush=True)
    print("bitwise equal:", torch.equal(ref[8].view(torch.int64), ref[12].view(torch.int64)))
_lib.call("oz_set_epilogue_warps", 12)
