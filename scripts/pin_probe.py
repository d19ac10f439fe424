import time, ctypes, torch
torch.cuda.init()
for mb in (64, 128, 256):
    t0 = time.perf_counter()
    x = torch.empty(mb * 2**20 // 4, dtype=torch.int32, pin_memory=True)
    t1 = time.perf_counter()
    d = torch.empty(mb * 2**20 // 4, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    t2 = time.perf_counter(); x.copy_(d, non_blocking=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    t4 = time.perf_counter(); x.copy_(d, non_blocking=True); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"{mb} MB: pinned alloc {1e3*(t1-t0):.1f} ms, D2H first {1e3*(t3-t2):.2f} ms ({mb/1024/(t3-t2):.1f} GB/s), again {1e3*(t5-t4):.2f} ms ({mb/1024/(t5-t4):.1f} GB/s)")
    del x
