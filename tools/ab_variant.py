"""K3 time per forced kernel variant (cta_group, tile N) for FP16 k-blocked and
FP8 configurations (results are bitwise identical across variants)."""
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from bench import gpu_inputs  # noqa: E402

f8, f16, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp16"), oz.get_format("fp32")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
only_defaults = len(sys.argv) > 2
A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
C = torch.empty((n, n), dtype=torch.float64, device="cuda")
for name, cfg in (("fp16 kb1024", oz.GemmConfig(f16, f32, k_block=1024)), ("fp8 kb1024", oz.GemmConfig(f8, f32, k_block=1024)),
                  ("fp8 defaults", oz.GemmConfig(f8, f32))):
    if only_defaults and name != "fp8 defaults":
        continue
    for rnd in range(2):
        for v in ((2, 192), (2, 128), (1, 128), (1, 64)):
            _lib.set_pair_variant(*v)
            oz.oz_gemm_device(A, B, cfg, out=C)
            ts = []
            for _ in range(2 if n >= 8192 else 10):
                _, st = oz.oz_gemm_device(A, B, cfg, out=C)
                ts.append(st.t_gemm * 1e3)
            h = hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:10]
            print(f"{name} variant {v}: K3 {min(ts):8.2f} ms C {h}", flush=True)
_lib.set_pair_variant(0, 0, 0)
