"""Golden vectors for the CLI, produced by running the REFERENCE CLI itself
(ozdgemm 1.0.0 from /root/reference/pkg/src; run in the container that has it):
    python tests/golden/gen_cli_golden.py
Writes cli.npz (gen_matrix streams, C dumps of `gemm` runs) and cli.json
(slices-table CSV text, the `gemm` reports minus timings)."""

from __future__ import annotations

import contextlib
import io
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from ozdgemm import cli as R  # noqa: E402

GEN_CASES = [(7, 9, 42, 1.0, 10.0), (9, 7, 42, 1.0, 10.0), (1, 1, 0, -1.0, 1.0), (33, 17, 2**40 + 5, 0.0, 8.0),
             (64, 64, 123456789, 1.0, 10.0)]
GEMM_CASES = [
    ["gemm", "--m", "16", "--n", "12", "--k", "64", "--type2", "fp8e4m3"],
    ["gemm", "--m", "8", "--n", "8", "--k", "32", "--type2", "fp16", "--type3", "fp32"],
    ["gemm", "--m", "10", "--n", "6", "--k", "40", "--type2", "fp16", "--kblock", "16", "--seed", "3"],
    ["gemm", "--m", "8", "--n", "8", "--k", "16", "--type2", "fp8e4m3", "--init", "powers2", "--seed", "9"],
    ["gemm", "--m", "12", "--n", "12", "--k", "24", "--type2", "fp8e4m3", "--fp64emu", "--max-slices", "4"],
]


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = R.main(argv)
    return code, buf.getvalue()


def main():
    arrays, meta = {}, {"gen": [], "gemm": []}
    for i, (r, c, seed, lo, hi) in enumerate(GEN_CASES):
        arrays[f"gen{i}"] = R.gen_matrix(r, c, seed, lo, hi).view(np.uint64)
        meta["gen"].append([r, c, seed, lo, hi])
    _, table = run(["slices-table"])
    meta["slices_table"] = table
    with tempfile.TemporaryDirectory() as td:
        for i, argv in enumerate(GEMM_CASES):
            dump = str(Path(td) / f"c{i}.npy")
            code, out = run(argv + ["--dump", dump])
            assert code == 0
            rep = json.loads(out)
            rep["stats"].pop("wall_s")
            rep.pop("wall_s_total")
            rep.pop("c_dump")
            arrays[f"c{i}"] = np.load(dump).view(np.uint64)
            meta["gemm"].append({"argv": argv, "report": rep})
    np.savez_compressed(HERE / "cli.npz", **arrays)
    (HERE / "cli.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print("wrote cli.npz, cli.json")


if __name__ == "__main__":
    main()
