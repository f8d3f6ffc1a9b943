import os, sys, json, subprocess, threading, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2509_17360_b200 import GpuCosineIndex
rows = bench.make_rows(1_000_000, 768)
idx = GpuCosineIndex(768, store_f32=True, store_bf16=True, capacity=rows.shape[0])
idx.insert_batch(np.arange(rows.shape[0]), rows, _checked=True)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
clk = []
stop = False
def sampler():
    while not stop:
        o = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        clk.append((time.time(), o)); time.sleep(0.05)
th = threading.Thread(target=sampler); th.start()
for b in (8, 1, 8, 16, 8):
    qs = bench.make_queries(rows, b, seed=100 + b)
    q = torch.from_numpy(qs).cuda()
    ids = torch.empty((b, 10), dtype=torch.int64, device="cuda"); sims = torch.empty((b, 10), dtype=torch.float64, device="cuda")
    cnt = torch.empty((b,), dtype=torch.int32, device="cuda"); cert = torch.zeros((b,), dtype=torch.uint8, device="cuda")
    for scan in ("fp32",):
        run = lambda: idx.query_device_cert(b, q.data_ptr(), 10, 0.9, ids.data_ptr(), sims.data_ptr(), cnt.data_ptr(), cert.data_ptr(), s.cuda_stream, scan=scan)
        run(); torch.cuda.synchronize()
        for g in range(6):
            t0 = time.time()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20): run()
            e1.record(); torch.cuda.synchronize()
            t1 = time.time()
            cs = [c for t, c in clk if t0 <= t <= t1]
            print(b, scan, g, round(e0.elapsed_time(e1) / 20, 4), int(cert.sum()), cs[:3], flush=True)
stop = True; th.join()
