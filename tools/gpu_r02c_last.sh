# Session 3 last check at HEAD: full GPU suite + smoke.
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_last.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_last.log
tail -3 gpurun_out/pytest_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
