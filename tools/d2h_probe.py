import torch, time
n = 3840*2160
d = torch.full((n,), -1, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
for rep in range(3):
    t0=time.perf_counter(); p = torch.empty(n, dtype=torch.int64, pin_memory=True); t1=time.perf_counter()
    p.copy_(d); torch.cuda.synchronize(); t2=time.perf_counter()
    print(f"alloc {1e3*(t1-t0):.2f} ms  copy {1e3*(t2-t1):.2f} ms  {n*8/(t2-t1)/1e9:.1f} GB/s")
p = torch.empty(n, dtype=torch.int64, pin_memory=True)
for rep in range(3):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); p.copy_(d, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print("event-timed pinned D2H", e0.elapsed_time(e1), "ms")
import numpy as np
h = np.empty(n, dtype=np.int64)
t0=time.perf_counter(); h[:] = p.numpy(); t1=time.perf_counter(); print("host memcpy", 1e3*(t1-t0))
t0=time.perf_counter(); x = d.cpu(); t1=time.perf_counter(); print("pageable .cpu()", 1e3*(t1-t0))
