"""cuBLAS bf16/fp16 GEMM for an ncu calibration of the tensor-pipe counters
(dev tool): what sm__pipe_tensor_cycles_active reads for a library GEMM at
the measured peak, beside the sweep's own reading."""
import torch
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    c = a @ b
ah, bh = a.half(), b.half()
for _ in range(3):
    c = ah @ bh
torch.cuda.synchronize()
