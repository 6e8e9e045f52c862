import sys, time, ctypes as C, numpy as np, torch
sys.path.insert(0, '.')
import paper_1407_4764_b200 as otf
from paper_1407_4764_b200 import _lib
dev = torch.device('cuda', 0); otf.set_device(0)
n, M, Q, K = 10_000_000, 16, 8, 256
x = torch.randn((n, M * Q), device=dev); x /= x.norm(dim=1, keepdim=True)
cents = torch.as_tensor(np.random.default_rng(9).standard_normal((M, K, Q)).astype(np.float32), device=dev)
codes = torch.empty((n, M), dtype=torch.uint8, device=dev)
lib = _lib.load(); st = torch.cuda.current_stream(dev); sp = C.c_void_p(st.cuda_stream)
def step():
    _lib.check(lib.otf_pq_encode(0, _lib.tptr(x), n, M * Q, _lib.tptr(cents), M, K, Q, _lib.tptr(codes), _lib.MEM_DEVICE, sp))
for _ in range(3): step()
torch.cuda.synchronize()
for i in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(st); step(); b.record(st); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step {i}: events {a.elapsed_time(b):.2f} ms, host call {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms")
    if i == 4: time.sleep(1.0)
