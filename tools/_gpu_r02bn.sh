cd $GRAFT_REPO_ROOT
TAG=r02bn
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/${TAG}_torchrun_w1.jsonl 2> gpurun_out/${TAG}_torchrun_w1.err; echo torchrun rc=$?; tail -3 gpurun_out/${TAG}_torchrun_w1.err; cut -c1-200 gpurun_out/${TAG}_torchrun_w1.jsonl
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
