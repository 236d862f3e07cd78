# round-2 GPU batch an: the driver's round-end sequence on the current tree (checkpoint)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2an_pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/r2an_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2an_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2an_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2an_ref.log 2>&1
