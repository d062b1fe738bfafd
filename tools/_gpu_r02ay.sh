cd $GRAFT_REPO_ROOT
TAG=r02ay
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum --clock-control none --csv python tools/cublas_pipe_probe.py > gpurun_out/${TAG}_cublas_pipe.csv 2>&1; echo rc=$?
