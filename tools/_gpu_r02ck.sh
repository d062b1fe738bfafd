# final build: launch list of a C2 bench run, reference arm, torchrun world 1
cd $GRAFT_REPO_ROOT
TAG=r02ck
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_l.log 2>&1; echo ncu launches rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_c2.jsonl 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/${TAG}_torchrun_w1.jsonl 2> gpurun_out/${TAG}_torchrun_w1.err; echo torchrun rc=$?
