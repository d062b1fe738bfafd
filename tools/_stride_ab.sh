# dev A/B: triangle sample stride / threshold rank at C2 (device ms/step and capture rows)
cd $GRAFT_REPO_ROOT
for cfg in ${CFGS:-"16 4" "16 5" "16 3" "20 4" "14 4"}; do
  set -- $cfg
  KNN_B200_TRI_STRIDE=$1 KNN_B200_TRI_RANK=$2 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('stride=$1 rank=$2', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'fallback_rows', d['gpu_stats']['fallback_rows'], 'rescored', d['gpu_stats']['rescored'], 'sm_mhz', d['clocks']['sm_mhz'])" >> gpurun_out/r01g_stride_ab.txt 2>&1
done
