cd $GRAFT_REPO_ROOT
TAG=r02bo
for v in bench.py bench_old.py bench.py bench_old.py; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29514 $v --gpus 1 --steps 5 --warmup 3 > gpurun_out/${TAG}_tmp.jsonl 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_tmp.jsonl').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1))" >> gpurun_out/${TAG}_ab.txt
done
