"""CUDA path vs the oracle (compiled reference when present, else the C
restatement), bit-exact, through the C ABI of libdisttrain_b200.so."""
import numpy as np
import pytest

import golden_cases as G
import parity_cases as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["intra", "select", "schedule", "exhaustive", "brute", "inter", "cost",
                                  "simulate", "stats", "disaggregated", "stream", "orchestration"])
def test_gpu_matches_oracle(name, gpu, oracle_best):
    rng = np.random.default_rng(4321 + len(name))
    getattr(P, "check_" + name)(gpu, oracle_best, rng)


@pytest.mark.parametrize("case", G.ALL, ids=lambda f: f.__name__)
def test_gpu_golden(case, gpu):
    case(gpu)


@pytest.mark.gpu
def test_gpu_stream_large_assembled_sums(gpu, oracle_best):
    """span 4 with samples of 16K-32K tokens: assembled microbatch sums above
    65535 (cost-table rows past the u16 token range) in intra+inter mode."""
    import numpy as np
    from parity_cases import H, assert_same
    from paper_2408_04275_b200.api import SampleBatch
    rng = np.random.default_rng(11)
    model, cluster, book = H.desk_model(), H.desk_cluster(64), H.desk_book()
    ci, co = gpu.cost_model(model, cluster, book), oracle_best.cost_model(model, cluster, book)
    n_batches, bs, dp, dp_me = 2, 1024, 16, 4
    pl = H.plan((1, dp_me, 1), (1, dp, 2), (1, dp_me, 1), bs)
    big = rng.random(n_batches * bs) < 0.5
    toks = np.where(big, rng.integers(16000, 32000, n_batches * bs),
                    rng.integers(1, 3000, n_batches * bs))
    s = SampleBatch.from_lists([(10, [int(t)]) for t in toks])
    ra = gpu.reorder_stream(ci, pl, s, n_batches, inter=True)
    rb = oracle_best.reorder_stream(co, pl, s, n_batches, inter=True)
    for k in ("output_order", "load_before", "load_after", "t_iter_before", "t_iter_after"):
        assert_same(ra[k], rb[k], k)


@pytest.mark.gpu
@pytest.mark.parametrize("inter", [False, True])
@pytest.mark.parametrize("pp", [(11, 3), (71, 7), (140, 3)])
def test_gpu_stream_many_stages(gpu, oracle_best, inter, pp):
    """Many-stage group simulations (p = 15 / 79 / 144 > 8 stages, vpp 1,
    span 2: register and shared-memory warp kernels), the shape of the plan
    model_orchestration picks for BASELINE config 5."""
    from parity_cases import H, assert_same
    from paper_2408_04275_b200.workload import synth_stream
    model, cluster, book = H.desk_model(), H.desk_cluster(1172), H.desk_book()
    ci, co = gpu.cost_model(model, cluster, book), oracle_best.cost_model(model, cluster, book)
    n_batches, bs = 3, 1024
    pl = H.plan((1, 8, 1), (1, 16, pp[0]), (1, 4, pp[1]), bs)
    s = synth_stream(n_batches * bs, seed=5, family="mixed")
    ra = gpu.reorder_stream(ci, pl, s, n_batches, inter=inter)
    rb = oracle_best.reorder_stream(co, pl, s, n_batches, inter=inter)
    for k in ("output_order", "load_before", "load_after", "t_iter_before", "t_iter_after"):
        assert_same(ra[k], rb[k], k)


@pytest.mark.gpu
def test_gpu_config5_chosen_plan(gpu, oracle_best):
    """BASELINE config 5: search the 72B MLLM on 1,172 GPUs at BS 16,384, then
    reorder (intra) a 16K-sample global batch with the chosen plan."""
    from parity_cases import H, assert_same
    from paper_2408_04275_b200.api import stats_to_c
    from paper_2408_04275_b200.workload import synth_stream
    m, cl, bk = H.mllm72b_model(), H.a800_cluster(1172), H.mllm72b_book()
    st = stats_to_c(m.seq_len, 2048.0, 2048.0)
    ci, co = gpu.cost_model(m, cl, bk), oracle_best.cost_model(m, cl, bk)
    g, r = gpu.model_orchestration(ci, st, 16384), oracle_best.model_orchestration(co, st, 16384)
    assert g["best"] == r["best"] and g["times"] == r["times"]
    s = synth_stream(16384, seed=1000, family="mixed")
    ra = gpu.reorder_stream(ci, g["best"], s, 1, inter=False)
    rb = oracle_best.reorder_stream(co, r["best"], s, 1, inter=False)
    for k in ("output_order", "load_before", "load_after", "t_iter_before", "t_iter_after"):
        assert_same(ra[k], rb[k], k)


@pytest.mark.gpu
def test_gpu_rejects_costs_outside_the_key_range(gpu):
    """A negative modality-token sum (Sample::valid never admits one,
    src/core.cpp:97) or one of 2^31 or more is reported, not misordered."""
    from parity_cases import H
    from paper_2408_04275_b200.api import InvalidArgument, SampleBatch
    model, cluster, book = H.desk_model(), H.desk_cluster(64), H.desk_book()
    ci = gpu.cost_model(model, cluster, book)
    pl = H.plan((1, 2, 1), (1, 2, 2), (1, 2, 1), 8)
    for bad in (-5, 2**30, 2**30):
        rows = [(1, [10]), (1, [bad, bad if bad > 0 else 0]), (1, [3])] + [(1, [7])] * 5
        s = SampleBatch.from_lists(rows)
        with pytest.raises(InvalidArgument):
            gpu.reorder_stream(ci, pl, s, 1, inter=False)
