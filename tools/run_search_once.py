"""model_orchestration for BASELINE config 3 (72B MLLM, 1172 GPUs, BS 1920),
twice (profiling driver; debug tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import helpers as H  # noqa: E402
from paper_2408_04275_b200 import native  # noqa: E402
from paper_2408_04275_b200.api import stats_to_c  # noqa: E402

pl = native.planner(0)
model = H.mllm72b_model()
cm = pl.cost_model(model, H.a800_cluster(1172), H.mllm72b_book())
st = stats_to_c(model.seq_len, 2048.0, 2048.0)
for _ in range(3):
    t0 = time.perf_counter()
    r = pl.model_orchestration(cm, st, 1920)
    print(f"{(time.perf_counter() - t0) * 1e3:.3f} ms", r["candidates_evaluated"], flush=True)
