import sys, hashlib
sys.path.insert(0, '/root/repo')
import torch
import paper_2508_00441_b200 as oz
from paper_2508_00441_b200 import _lib
from bench import gpu_inputs
n = 8192
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
for cut in (None, 11):
    cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), fp64_emulation=True, pair_cutoff=cut)
    for rnd in range(2):
        for v in ((2, 128), (1, 128), (1, 64)):
            _lib.set_pair_variant(*v)
            oz.oz_gemm_device(A, B, cfg, out=C)
            _, st = oz.oz_gemm_device(A, B, cfg, out=C)
            print(f"emu cut={cut} {v}: K3 {st.t_gemm*1e3:8.2f} ms", flush=True)
