"""brute_force_oracle on the GPU vs the CPU reference at 32/64/128 GPUs
(timing tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import helpers as H  # noqa: E402
import oracle  # noqa: E402
from paper_2408_04275_b200 import native  # noqa: E402
from paper_2408_04275_b200.api import stats_to_c  # noqa: E402

pl = native.planner(0)
ora, kind = oracle.best()
for n in (32, 64, 128):
    model, cluster, book = H.desk_model(), H.desk_cluster(n), H.desk_book()
    st = stats_to_c(model.seq_len, 1000.0, 1000.0)
    cg, co = pl.cost_model(model, cluster, book), ora.cost_model(model, cluster, book)
    pl.brute_force_oracle(cg, st, 256, 1, n)
    t0 = time.perf_counter()
    a = pl.brute_force_oracle(cg, st, 256, 1, n)
    dg = time.perf_counter() - t0
    print(n, "GPU", f"{dg * 1e3:.2f} ms", a["candidates_evaluated"],
          f"{a['candidates_evaluated'] / dg:.3g} plans/s", flush=True)
    if n <= 64:
        t0 = time.perf_counter()
        b = ora.brute_force_oracle(co, st, 256, 1, n)
        dc = time.perf_counter() - t0
        print("   CPU", kind, f"{dc * 1e3:.2f} ms", f"{b['candidates_evaluated'] / dc:.3g} plans/s",
              "bit-exact" if a == b else "MISMATCH", flush=True)
