# final-build evidence (packed-fold build): GPU suite, smoke, bench (C2), reference arm, torchrun world 1,
# launch list, C3/C4 steps, C3 sharded emulation at 8 ranks, ncu --set full of the C3 band rescore
cd $GRAFT_REPO_ROOT
TAG=r02ca
timeout 2000 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; cut -c1-250 gpurun_out/${TAG}_bench_c2.jsonl
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_c2.jsonl 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29516 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/${TAG}_torchrun_w1.jsonl 2> gpurun_out/${TAG}_torchrun_w1.err; echo torchrun rc=$?
for c in "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
  echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_l.log 2>&1; echo ncu launches rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:rescore_capture_kernel -c 1 -o gpurun_out/${TAG}_band_c3 python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > gpurun_out/${TAG}_ncu_band.log 2>&1; echo ncu band rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore" --csv python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/${TAG}_c2_rescore.csv 2>&1; echo c2 ncu rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore_capture" --csv python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > gpurun_out/${TAG}_c3_rescore.csv 2>&1; echo c3 ncu rc=$?
