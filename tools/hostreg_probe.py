"""Dev probe: cost of cudaHostRegister/Unregister on a pageable 1 GB buffer,
whole and in parallel slices, and the DMA rate from registered memory."""
import ctypes, threading, time
import numpy as np
import torch

torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12") if False else None
import glob, os
cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
        glob.glob("/usr/local/cuda/lib64/libcudart.so*")
rt = ctypes.CDLL(cands[0])
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
nbytes = 1024 * 1000 * 1000
x = np.ones(nbytes // 4, dtype=np.float32)
p = x.ctypes.data
d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
for rep in range(3):
    t0 = time.perf_counter(); rc = rt.cudaHostRegister(p, nbytes, 0); t1 = time.perf_counter()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(torch.from_numpy(x), non_blocking=True); e.record(); torch.cuda.synchronize()
    t2 = time.perf_counter(); rc2 = rt.cudaHostUnregister(p); t3 = time.perf_counter()
    print(f"whole: register {1e3*(t1-t0):.1f} ms rc={rc}, dma {s.elapsed_time(e):.1f} ms, unregister {1e3*(t3-t2):.1f} ms rc={rc2}")
for nt in (4, 8, 12, 16):
    page = 4096
    base = (p + page - 1) // page * page
    usable = (p + nbytes) // page * page - base
    sl = usable // nt // page * page
    rcs = [0] * nt
    def reg(i):
        rcs[i] = rt.cudaHostRegister(base + i * sl, sl if i < nt - 1 else usable - i * sl, 0)
    def unreg(i):
        rt.cudaHostUnregister(base + i * sl)
    t0 = time.perf_counter(); th = [threading.Thread(target=reg, args=(i,)) for i in range(nt)]
    [t.start() for t in th]; [t.join() for t in th]; t1 = time.perf_counter()
    th = [threading.Thread(target=unreg, args=(i,)) for i in range(nt)]
    t2 = time.perf_counter(); [t.start() for t in th]; [t.join() for t in th]; t3 = time.perf_counter()
    print(f"{nt} threads: register {1e3*(t1-t0):.1f} ms rcs={set(rcs)}, unregister {1e3*(t3-t2):.1f} ms")
