import torch, time, numpy as np, ctypes
x = np.random.rand(9_000_000)
d = torch.empty(9_000_000, dtype=torch.float64, device="cuda")
for mode in ("pageable", "pinned"):
    src = torch.from_numpy(x)
    if mode == "pinned":
        src = src.pin_memory()
    for r in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for k in range(8):
            d.copy_(src, non_blocking=(mode=="pinned"))
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(mode, f"{8*72e6/dt/1e9:.1f} GB/s")
t=time.perf_counter(); p = torch.from_numpy(x).pin_memory(); print("pin_memory copy 72MB", time.perf_counter()-t)
cudart = ctypes.CDLL("libcudart.so")
