cd $GRAFT_REPO_ROOT
TAG=r02bz
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rfE -k "edge_shapes or golden or random" > gpurun_out/${TAG}_pytest_edge.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_edge.log
for i in 1 2; do timeout 300 python tools/profile_solve.py --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/${TAG}_c2_first.txt 2>&1; done
timeout 900 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section SchedulerStats --section WarpStateStats --section Occupancy --section InstructionStats --clock-control none -k regex:exact_fused -c 1 python tools/profile_solve.py --n 131072 --d 256 --k 10 --arith exact --seed 1 --reps 1 > gpurun_out/${TAG}_exact_ncu.txt 2>&1; echo ncu rc=$?
