cd $GRAFT_REPO_ROOT
TAG=r02bg
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/${TAG}_torchrun_w1.jsonl 2> gpurun_out/${TAG}_torchrun_w1.err; echo torchrun rc=$?; cut -c1-300 gpurun_out/${TAG}_torchrun_w1.jsonl
