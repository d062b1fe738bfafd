cd $GRAFT_REPO_ROOT
TAG=r02be
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cli.py tests/test_f64_accum.py -q -rfE -x > gpurun_out/${TAG}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest.log
for i in 1 2; do timeout 300 ./build/bench_dropin 1000000 256 10 1 5 1 >> gpurun_out/${TAG}_dropin.txt 2>&1; done; echo dropin rc=$?; tail -2 gpurun_out/${TAG}_dropin.txt
