"""One default-mode (intra + inter) disaggregated_reorder over a 128-batch
slice of the BASELINE config 4 stream (profiling driver; debug tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import helpers as H  # noqa: E402
from paper_2408_04275_b200 import native  # noqa: E402
from paper_2408_04275_b200.workload import synth_stream  # noqa: E402

pl = native.planner(0)
cm = pl.cost_model(H.desk_model(), H.desk_cluster(1172), H.desk_book())
plan = H.plan((1, 128, 1), (1, 128, 2), (1, 128, 1), 16384)
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = synth_stream(nb * 16384, 1000, "mixed")
r = pl.reorder_stream(cm, plan, s, nb, inter=True)
print("ok", r["t_iter_after"][:2])
