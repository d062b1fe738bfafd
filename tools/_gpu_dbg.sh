(CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/_dbg_nccl2.py 2>&1 | grep -v "^NCCL") > gpurun_out/r02r_dbg.log
(CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/_dbg_nccl2.py nobcast 2>&1 | grep -v "^NCCL") >> gpurun_out/r02r_dbg.log
