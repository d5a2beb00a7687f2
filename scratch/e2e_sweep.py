import ctypes as C, os, sys, time, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
G, N, D = 64, 65536, 128
p = _abi.make_problem(G, N, D, "bf16")
pin = dict(dtype=torch.bfloat16, pin_memory=True)
hq = torch.randn(G, N, D).bfloat16().pin_memory(); hk = hq.clone().pin_memory()
hq /= hq.float().norm(dim=-1, keepdim=True).bfloat16(); hk.copy_(hq)
hv = torch.rand(G, D, N).bfloat16().pin_memory(); hw = hv.clone().pin_memory()
hout = torch.empty((G, D, N), **pin); hdq = torch.empty((G, N, D), **pin); hdk = torch.empty((G, D, N), **pin); hdv = torch.empty((G, D, N), **pin)
hg = torch.empty((G, N), dtype=torch.float32, pin_memory=True)
err = _abi.ErrorInfo()
def step():
    st = L.la_host_step(C.byref(p), hq.data_ptr(), 1, hk.data_ptr(), 1, hv.data_ptr(), 0, hw.data_ptr(), 0,
                        hout.data_ptr(), hg.data_ptr(), hdq.data_ptr(), hdk.data_ptr(), hdv.data_ptr(), C.byref(err))
    assert st == 0, err.message
step()
t = time.perf_counter()
for _ in range(3): step()
print(os.environ.get("LA_HOST_BLOCKS"), (time.perf_counter() - t) / 3 * 1e3, "ms")
