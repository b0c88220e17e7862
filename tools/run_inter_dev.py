"""Default-mode disaggregated_reorder over the whole config-4 stream through
the DEVICE entry point (one launch per kernel, all 1024 batches): the
inter kernel at full occupancy (profiling driver; debug tool)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import helpers as H  # noqa: E402
from paper_2408_04275_b200 import _capi as A  # noqa: E402
from paper_2408_04275_b200 import native  # noqa: E402
from paper_2408_04275_b200.workload import synth_stream  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pl = native.planner(0)
cm = pl.cost_model(H.desk_model(), H.desk_cluster(1172), H.desk_book())
plan = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384).to_c()
s = synth_stream(nb * 16384, 1000, "mixed")
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
d = [dev(s.image_offsets), dev(s.image_tokens), dev(s.audio_offsets), dev(s.audio_tokens)]
ds = A.Samples(s.n, None, *[C.cast(x.data_ptr(), C.POINTER(C.c_int32)) for x in d])
outs = [torch.empty(s.n, dtype=torch.int32, device="cuda"),
        torch.empty(nb * 128, dtype=torch.float64, device="cuda"),
        torch.empty(nb * 128, dtype=torch.float64, device="cuda"),
        torch.empty(nb, dtype=torch.float64, device="cuda"),
        torch.empty(nb, dtype=torch.float64, device="cuda"),
        torch.empty(nb, dtype=torch.uint8, device="cuda")]
mode = A.ReorderMode(1, 1, 0)
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pl._check(pl.lib.reorder_stream_dev(pl.ctx, cm.h, C.byref(plan), C.byref(mode), C.byref(ds),
                                        nb, *[C.c_void_p(x.data_ptr()) for x in outs], None))
    e1.record()
    torch.cuda.synchronize()
    print(f"step {it}: {e0.elapsed_time(e1):.3f} ms", flush=True)
