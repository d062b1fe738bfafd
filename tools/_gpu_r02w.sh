timeout 2400 python -m pytest tests -m gpu -q -rfE --durations=10 > gpurun_out/r02w_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r02w_bench.jsonl 2>gpurun_out/r02w_bench.err
