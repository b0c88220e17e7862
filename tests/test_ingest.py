"""Trace ingest (ingest_trace, src/workload.cpp:115-153).

CPU (not gpu): the parser of csrc/jsonl.cuh compiled for the host by a test
harness (tests/native/jsonl_host.cpp) is fuzzed line by line against the
compiled reference, and its number conversion against nlohmann itself
(tests/native/json_ref.cpp); the reference's own ingest tests
(tests/test_workload.cpp:98-133) pin the oracle.
GPU: dtb_ingest_trace (the CUDA path) against the compiled reference on whole
traces — CSR arrays identical, errors with the same kind and line.
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

import trace_cases as TC

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2408_04275_b200", "csrc")
NATIVE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "native")
BUILD = os.path.join(ROOT, "build", "tests")


def _json_inc():
    for s in sys.path:
        p = os.path.join(s, "include", "cudnn_frontend", "thirdparty")
        if os.path.isdir(os.path.join(p, "nlohmann")):
            return p
    return None


def _build(name, src, extra=()):
    os.makedirs(BUILD, exist_ok=True)
    out = os.path.join(BUILD, name)
    deps = [src, os.path.join(CSRC, "jsonl.cuh"), os.path.join(CSRC, "jsonl_tables.cuh")]
    if not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-I" + CSRC,
                               *extra, src, "-o", out])
    return C.CDLL(out)


@pytest.fixture(scope="module")
def host_parser():
    lib = _build("libjsonl_host.so", os.path.join(NATIVE, "jsonl_host.cpp"))
    lib.jh_parse.argtypes = [C.c_char_p, C.c_int, C.c_longlong, C.POINTER(C.c_longlong),
                             C.POINTER(C.c_int), C.c_int]
    lib.jh_number.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_longlong)]
    return lib


@pytest.fixture(scope="module")
def nlohmann_ref():
    inc = _json_inc()
    if inc is None:
        pytest.skip("nlohmann/json header not found")
    lib = _build("libjson_ref.so", os.path.join(NATIVE, "json_ref.cpp"), ["-I" + inc])
    lib.jref_number.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_longlong)]
    return lib


# J_* of csrc/jsonl.cuh
J_OK, J_BLANK, J_PARSE, J_INVARIANT, J_UNSUPPORTED = range(5)


def host_parse(lib, line: bytes, cap: int):
    out = (C.c_longlong * 6)()
    vals = (C.c_int * 4096)()
    st = lib.jh_parse(line, len(line), cap, out, vals, 4096)
    if st != J_OK:
        return st, None
    ni, na = out[3], out[4]
    return st, (out[2], list(vals[:ni]), list(vals[ni:ni + na]))


def ref_parse(ref, line: bytes, cap: int):
    """The reference on a one-line trace -> (status, record)."""
    from paper_2408_04275_b200 import api
    try:
        b = ref.ingest_trace(line, cap)
    except api.TraceError as e:
        assert e.line() == 1
        return (J_PARSE if e.kind() == "ParseError" else J_INVARIANT), None
    except api.InvalidArgument:
        return J_UNSUPPORTED, None
    if b.n == 0:
        return J_BLANK, None
    assert b.n == 1
    return J_OK, (int(b.text[0]), b.image_tokens.tolist(), b.audio_tokens.tolist())


# ---------------------------------------------------------------- oracle pins
def test_reference_ingest_known_answers(ref):
    """tests/test_workload.cpp:98-121 on the compiled reference."""
    from paper_2408_04275_b200 import api
    assert ref.ingest_trace(b"", 8192).n == 0
    with pytest.raises(api.TraceError) as e:
        ref.ingest_trace(b'{"text_tokens": 5}\nnot json\n', 8192)
    assert e.value.line() == 2 and e.value.kind() == "ParseError"
    with pytest.raises(api.TraceError) as e:
        ref.ingest_trace(b'{"text_tokens": 5, "image_subseqs": [-3]}\n', 8192)
    assert e.value.line() == 1 and e.value.kind() == "InvariantViolation"


def test_reference_round_trip(ref):
    """tests/test_workload.cpp:123-133: write_trace -> ingest_trace is exact."""
    from paper_2408_04275_b200.workload import synth_stream
    batch = synth_stream(256, seed=3)
    back = ref.ingest_trace(TC.write_trace(batch), 8192)
    for a in ("text", "image_offsets", "image_tokens", "audio_offsets", "audio_tokens"):
        np.testing.assert_array_equal(getattr(back, a), getattr(batch, a))


# ------------------------------------------------------- host-compiled parser
def test_number_conversion_matches_nlohmann(host_parser, nlohmann_ref):
    import random
    rng = random.Random(7)
    forms = list(TC.NUMBER_FORMS) + [TC.random_number(rng) for _ in range(30000)]
    for s in forms:
        b = s.encode()
        v1, v2 = C.c_longlong(), C.c_longlong()
        r1 = host_parser.jh_number(b, len(b), C.byref(v1))
        r2 = nlohmann_ref.jref_number(b, len(b), C.byref(v2))
        if r2 == 1:  # nlohmann rejects: malformed (-1 here) or overflow (1)
            assert r1 in (-1, 1), s
        else:
            assert r2 == 0 and r1 == 0 and v1.value == v2.value, (s, v1.value, v2.value)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_line_parser_matches_reference(host_parser, ref, seed):
    lines = TC.random_lines(seed, 3000)
    kinds = {}
    for line in lines:
        for cap in (8192, 1 << 62):
            got = host_parse(host_parser, line, cap)
            want = ref_parse(ref, line, cap)
            assert got == want, (line, cap, got, want)
            kinds[got[0]] = kinds.get(got[0], 0) + 1
    # the generator reaches every outcome
    assert all(kinds.get(k, 0) > 0 for k in (J_OK, J_BLANK, J_PARSE, J_INVARIANT)), kinds


def test_line_parser_edge_cases(host_parser, ref):
    cases = [
        b'{"text_tokens": 1, "text_tokens": 2}', b'{"text_\\u0074okens": 7}',
        b'\xef\xbb\xbf{"text_tokens": 7}', b' \xef\xbb\xbf{"text_tokens": 7}', b'\xef\xbb{"a":1}',
        b'{"text_tokens": 7}\r', b'{"text_tokens": true}', b'{"text_tokens": null}',
        b'{"text_tokens": 5, "image_subseqs": [true]}', b'{"text_tokens": 5, "image_subseqs": {}}',
        b'{"text_tokens": 5, "image_subseqs": null}', b'{"text_tokens": 5, "x": "\\ud800"}',
        b'{"text_tokens": 5, "x": "\\ud800\\udc00"}', b'{"text_tokens": 5, "x": "\\udc00"}',
        b'{"text_tokens": 5, "x": "\xc0\xaf"}', b'{"text_tokens": 5, "x": "\xed\xa0\x80"}',
        b'{"text_tokens": 5, "x": "\xf4\x90\x80\x80"}', b'{"text_tokens": 5, "x": "\xf0\x9f\x98\x80"}',
        b'{"text_tokens": 5, "x": "\x1f"}', b'{"text_tokens": 5, "x": "\x7f"}',
        b'{"text_tokens": 0}', b'{"text_tokens": 0, "image_subseqs": [0]}',
        b'{"text_tokens": 8192}', b'{"text_tokens": 8193}', b'{"text_tokens": -1}',
        b'{"text_tokens": 1, "audio_subseqs": [-1]}', b'{"text_tokens": 1e300}',
        b'{"text_tokens": 4611686018427387904, "image_subseqs": [4611686018427387904, '
        b'4611686018427387904, 4611686018427387904, 5]}',
        b'{"text_tokens": 18446744073709551615, "image_subseqs": [2]}',
        b'{"text_tokens": 5, "y": ' + b"[" * 1100 + b"]" * 1100 + b"}",
        b'{"text_tokens": 5, "y": ' + b"[" * 900 + b"]" * 900 + b"}",
        b'[{"text_tokens": 5}]', b'{"a": {"text_tokens": 5}}', b'{"text_tokens": 5}}',
        b'{"text_tokens" 5}', b'{"text_tokens": 5 "image_subseqs": []}', b'{"text_tokens": 05}',
        b'{"text_tokens": 5, "image_subseqs": [1,]}', b'{"text_tokens": 5, "image_subseqs": [,1]}',
        b'{"text_tokens": 2.5, "image_subseqs": [0.9999999999999999999]}',
        b'{"text_tokens": 5, "image_subseqs": [1e-400, -0.0, -0.5]}',
    ]
    for line in cases:
        got = host_parse(host_parser, line, 8192)
        want = ref_parse(ref, line, 8192)
        if got[0] == J_UNSUPPORTED and want[0] == J_OK:
            continue  # nesting beyond this ABI's limit (documented)
        assert got == want, (line, got, want)


# ------------------------------------------------------------------ GPU path
def _assert_same_ingest(gpu, ref, data: bytes, cap: int):
    from paper_2408_04275_b200 import api
    try:
        want = ref.ingest_trace(data, cap)
        werr = None
    except (api.TraceError, api.InvalidArgument) as e:
        want, werr = None, e
    try:
        got = gpu.ingest_trace(data, cap)
        gerr = None
    except (api.TraceError, api.InvalidArgument) as e:
        got, gerr = None, e
    if werr is not None:
        assert gerr is not None and type(gerr) is type(werr), (gerr, werr)
        if isinstance(werr, api.TraceError):
            assert (gerr.kind(), gerr.line()) == (werr.kind(), werr.line())
        return
    assert gerr is None, gerr
    for a in ("text", "image_offsets", "image_tokens", "audio_offsets", "audio_tokens"):
        np.testing.assert_array_equal(getattr(got, a), getattr(want, a), err_msg=a)


@pytest.mark.gpu
def test_gpu_ingest_known_answers(gpu, ref):
    for data in (b"", b"\n", b"\n\n  \r\n", b'{"text_tokens": 5}\nnot json\n',
                 b'{"text_tokens": 5, "image_subseqs": [-3]}\n', b'{"text_tokens": 5}',
                 b'{"text_tokens": 5}\r\n\r\n{"text_tokens": 6, "audio_subseqs": [7]}'):
        _assert_same_ingest(gpu, ref, data, 8192)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 2])
def test_gpu_ingest_random_lines(gpu, ref, seed):
    """Whole traces of fuzzed lines: the first failing line decides."""
    lines = TC.random_lines(seed, 4000)
    good = [ln for ln in lines if ref_parse(ref, ln, 8192)[0] in (J_OK, J_BLANK)]
    _assert_same_ingest(gpu, ref, b"\n".join(good) + b"\n", 8192)
    _assert_same_ingest(gpu, ref, b"\n".join(good), 8192)  # no trailing newline
    for k in range(12):  # one bad line somewhere
        import random
        rng = random.Random(seed * 100 + k)
        bad = [ln for ln in lines if ref_parse(ref, ln, 8192)[0] in (J_PARSE, J_INVARIANT)]
        mix = list(good)
        for _ in range(rng.randint(1, 3)):
            mix.insert(rng.randint(0, len(mix)), rng.choice(bad))
        _assert_same_ingest(gpu, ref, b"\n".join(mix), 8192)


@pytest.mark.gpu
def test_gpu_ingest_synthetic_stream(gpu, ref):
    """write_trace of a 200K-sample mixed stream round-trips exactly."""
    from paper_2408_04275_b200.workload import synth_stream
    batch = synth_stream(200_000, seed=5)
    data = TC.write_trace(batch)
    got = gpu.ingest_trace(data, 8192)
    for a in ("text", "image_offsets", "image_tokens", "audio_offsets", "audio_tokens"):
        np.testing.assert_array_equal(getattr(got, a), getattr(batch, a), err_msg=a)
    _assert_same_ingest(gpu, ref, data[:2_000_000], 8192)
