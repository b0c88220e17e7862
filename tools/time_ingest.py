"""Times dtb_ingest_trace_dev (device bytes -> device CSR) on a write_trace
JSONL stream, and the reference's ingest_trace (1 thread) on a slice.
usage: python tools/time_ingest.py [n_samples_millions]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import trace_cases as TC
from paper_2408_04275_b200 import native
from paper_2408_04275_b200.workload import synth_stream

m = float(sys.argv[1]) if len(sys.argv) > 1 else 16
base_n = 1 << 20
base = TC.write_trace(synth_stream(base_n, seed=1))
reps = max(1, int(round(m * (1 << 20) / base_n)))
data = base * reps
n = base_n * reps
print(f"trace: {n} samples, {len(data) / 1e6:.1f} MB", flush=True)
gpu = native.planner()
d = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
res = gpu.ingest_trace_dev(d.data_ptr(), len(data), 8192)
assert res.n_samples == n, res.n_samples
o = dict(cap_samples=n, cap_image=res.n_image, cap_audio=res.n_audio)
bufs = dict(text_tokens=torch.empty(n, dtype=torch.int32, device="cuda"),
            image_offsets=torch.empty(n + 1, dtype=torch.int32, device="cuda"),
            image_tokens=torch.empty(max(1, res.n_image), dtype=torch.int32, device="cuda"),
            audio_offsets=torch.empty(n + 1, dtype=torch.int32, device="cuda"),
            audio_tokens=torch.empty(max(1, res.n_audio), dtype=torch.int32, device="cuda"))
o.update({k: v.data_ptr() for k, v in bufs.items()})
for _ in range(2):
    gpu.ingest_trace_dev(d.data_ptr(), len(data), 8192, o)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    gpu.ingest_trace_dev(d.data_ptr(), len(data), 8192, o)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
t = min(ts)
b = synth_stream(base_n, seed=1)
assert np.array_equal(bufs["text_tokens"][:base_n].cpu().numpy(), b.text)
assert np.array_equal(bufs["image_tokens"][:len(b.image_tokens)].cpu().numpy(), b.image_tokens)
print(f"gpu ingest_trace_dev: {t * 1e3:.2f} ms  {len(data) / t / 1e9:.1f} GB/s  "
      f"{n / t / 1e6:.0f} M samples/s", flush=True)
import oracle
if oracle.ref_available():
    ref = oracle.ref()
    sl = base[: len(base) // 4]
    sl = sl[: sl.rindex(b"\n") + 1]
    t0 = time.perf_counter()
    r = ref.ingest_trace(sl, 8192)
    tr = time.perf_counter() - t0
    print(f"reference ingest_trace (1 thread): {r.n / tr / 1e6:.2f} M samples/s "
          f"{len(sl) / tr / 1e6:.1f} MB/s")
