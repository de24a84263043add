import time, torch, numpy as np, paper_1903_00227_b200 as wrs
n, k = 10**8, 10**9
Wd = wrs.Weights.generate_range("uniform", 0.0, n, 0, n, 42)
hw = torch.empty(n, dtype=torch.float64, pin_memory=True); hw.numpy()[:] = Wd.values(); Wd.free()
ho = torch.empty(k, dtype=torch.int32, pin_memory=True)
for it in range(4):
    torch.cuda.synchronize(); t0=time.perf_counter()
    W = wrs.Weights.from_array(hw.numpy()); t1=time.perf_counter()
    S = wrs.Sampler.build(W, "psa", 1); t2=time.perf_counter()
    S.draw_into(42, k, 1, ho.data_ptr()); t3=time.perf_counter()
    S.free(); W.free(); t4=time.perf_counter()
    print(f"from_array {1e3*(t1-t0):.1f} build {1e3*(t2-t1):.1f} draw {1e3*(t3-t2):.1f} free {1e3*(t4-t3):.1f} total {1e3*(t3-t0):.1f} ms")
