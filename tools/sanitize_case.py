"""Small multi-wave Ozaki GEMMs for compute-sanitizer (memcheck / racecheck /
synccheck): 2048 x 2048 x 256 — 88 CTA-pair tiles of 256 x 192 for 74 units,
so the persistent loop runs two tile waves — in the default, 1-CTA 128 x 64,
emulated and fixed-step grouped variants, each checked bitwise against the
first.  usage: python tools/sanitize_case.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from bench import gpu_inputs  # noqa: E402

A, _ = gpu_inputs(torch, 2048, 256, 8, 0.5, 1000, "cuda")
_, B = gpu_inputs(torch, 8, 256, 2048, 0.5, 2000, "cuda")
f8, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp32")
ref = None
for name, variant, kw in (("defaults 2x192", (2, 192), {}), ("defaults 1x64", (1, 64), {}),
                          ("emu 2x128", (2, 128), {"fp64_emulation": True}),
                          ("fixed cut 9 2x192", (2, 192), {"pair_cutoff": 9, "slice_exponents": "fixed"})):
    _lib.set_pair_variant(*variant)
    C, st = oz.oz_gemm_device(A, B, oz.GemmConfig(f8, f32, **kw))
    torch.cuda.synchronize()
    if ref is None:
        ref = C.clone()
    same = torch.equal(C.view(torch.int64), ref.view(torch.int64)) if "fixed" not in name else "n/a (own semantics)"
    print(f"{name}: pairs {st.gemm_count} bitwise == defaults: {same}", flush=True)
_lib.set_pair_variant(0, 0, 0)
