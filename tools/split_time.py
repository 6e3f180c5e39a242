"""Device time of the row split (adaptive vs fixed) for rows x kb operands.
usage: split_time.py rows kb"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200.slicing import split_deferred  # noqa: E402
from bench import gpu_inputs  # noqa: E402

rows, kb = int(sys.argv[1]), int(sys.argv[2])
X, _ = gpu_inputs(torch, rows, kb, 8, 0.5, 1000, "cuda")
f = oz.get_format("fp8e4m3")
params = oz.compute_params(53, f.mant_bits, 24, kb)
for name, kw in (("adaptive", {}), ("fixed12", {"fixed": True, "max_planes": 12})):
    for rep in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        ds = split_deferred(X, f, params, False, **kw)
        e[1].record()
        torch.cuda.synchronize()
        print(f"{name} rows={rows} kb={kb}: {e[0].elapsed_time(e[1]):.2f} ms s={ds.sf.cpu().tolist()}")
        del ds
