# dev A/B: rescore_kernel register budget (KNN_RESCORE_MINB 3 vs 2) -- kernel time under ncu and bench step
cd $GRAFT_REPO_ROOT
for minb in 3 2 4; do
  if [ $minb != 3 ]; then
    touch paper_0906_0231_b200/csrc/tensor_path.cu
    make lib NVCC=/usr/local/cuda/bin/nvcc NVFLAGS_EXTRA=-DKNN_RESCORE_MINB=$minb > /dev/null 2>&1 || echo "build $minb failed"
  fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rescore_kernel --csv python tools/profile_solve.py --n 1000000 --reps 2 2>/dev/null | grep gpu__time_duration | sed "s/^/minb=$minb /" >> gpurun_out/r01k_rescore_ab.txt
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('minb=$minb bench', round(d['ms_per_step'],2))" >> gpurun_out/r01k_rescore_ab.txt
done
