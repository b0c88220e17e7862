"""Trace-JSONL inputs for the ingest parity tests (ingest_trace,
src/workload.cpp:115-153): seeded random records in write_trace's format and
hand-written / randomly mutated lines that exercise the JSON grammar, the
int64 conversion and Sample::valid."""
import json
import random

import numpy as np

NUMBER_FORMS = [
    "0", "-0", "7", "-7", "01", "1.", ".5", "-", "+1", "1e", "1e+", "1.5e3", "2.9999999999999999999",
    "3.0", "-0.0", "0.1", "0.9999999999999999999", "0.99999999999999994", "0.99999999999999995",
    "9223372036854775807", "9223372036854775808", "-9223372036854775808", "-9223372036854775809",
    "18446744073709551615", "18446744073709551616", "9223372036854775807.0", "9223372036854774784.0",
    "9223372036854775295.9", "9223372036854775296", "4503599627370495.5", "4503599627370496.5",
    "4503599627370497.5", "9007199254740993", "9007199254740993.0", "9007199254740993.0000001",
    "9007199254740995", "1e19", "1e20", "1e300", "1e308", "1.7976931348623157e308",
    "1.7976931348623158e308", "1.7976931348623159e308", "1e309", "1e400", "-1e400", "1e-400",
    "123456789012345678901234567890", "0.000000000000000000001e21", "1E2", "1e+2", "1e-2",
    "100e-2", "12.5e-1", "0e0", "0e999999999999", "5e-324", "1e-99999999999999",
]


def random_number(rng: random.Random) -> str:
    k = rng.random()
    if k < 0.3:
        return rng.choice(NUMBER_FORMS)
    if k < 0.55:
        return str(rng.randint(-10 ** rng.randint(0, 21), 10 ** rng.randint(0, 21)))
    sign = "-" if rng.random() < 0.3 else ""
    ip = rng.choice(["0", str(rng.randint(1, 10 ** rng.randint(1, 20)))])
    s = sign + ip
    if rng.random() < 0.7:
        frac = "".join(rng.choice("0123456789" if rng.random() < 0.5 else "09")
                       for _ in range(rng.randint(1, 30)))
        s += "." + frac
    if rng.random() < 0.5:
        s += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.randint(0, 330))
    return s


def _ws(rng):
    return rng.choice(["", "", "", " ", "  ", "\t", " \r "])


def _value(rng, depth=0):
    k = rng.random()
    if depth > 3 or k < 0.3:
        return random_number(rng)
    if k < 0.4:
        return rng.choice(["true", "false", "null"])
    if k < 0.55:
        return json.dumps(rng.choice(["x", "é", "a\\b", "☃", "\U0001F600", ""]))
    if k < 0.75:
        return "[" + ",".join(_ws(rng) + _value(rng, depth + 1) for _ in range(rng.randint(0, 3))) + "]"
    keys = [rng.choice(["a", "text_tokens", "b c", "image_subseqs"]) for _ in range(rng.randint(0, 3))]
    return "{" + ",".join(json.dumps(kk) + ":" + _value(rng, depth + 1) for kk in keys) + "}"


def _int_list(rng, lo=0, hi=3000):
    return [rng.randint(lo, hi) for _ in range(rng.randint(0, 4))]


def random_record(rng: random.Random) -> str:
    """One line: mostly well-formed records with variations in layout."""
    fields = [("text_tokens", str(rng.randint(0, 2000)))]
    if rng.random() < 0.8:
        fields.append(("image_subseqs", "[" + ",".join(map(str, _int_list(rng))) + "]"))
    if rng.random() < 0.4:
        fields.append(("audio_subseqs", "[" + ",".join(map(str, _int_list(rng))) + "]"))
    r = rng.random()
    if r < 0.15:  # numbers of every form in the token fields
        fields = [(k, random_number(rng) if k == "text_tokens" else
                   "[" + ",".join(random_number(rng) for _ in range(rng.randint(0, 3))) + "]")
                  for k, _ in fields]
    elif r < 0.25:  # extra keys / nested values
        fields.insert(rng.randint(0, len(fields)), (rng.choice(["meta", "id", "x"]), _value(rng)))
    elif r < 0.32:  # duplicate keys (last wins)
        k, _ = rng.choice(fields)
        fields.append((k, str(rng.randint(0, 50)) if k == "text_tokens" else "[1, 2]"))
    elif r < 0.38:  # wrong types
        k, _ = rng.choice(fields)
        fields = [(kk, _value(rng) if kk == k else vv) for kk, vv in fields]
    elif r < 0.42:  # escaped keys
        fields = [(k.replace("t", "\\u0074", 1), v) for k, v in fields]
    elif r < 0.45:  # missing text_tokens
        fields = fields[1:]
    rng.shuffle(fields)
    body = "{" + ",".join(_ws(rng) + json.dumps(k).replace("\\\\u0074", "\\u0074") + _ws(rng) + ":" +
                          _ws(rng) + v + _ws(rng) for k, v in fields) + "}"
    body = _ws(rng) + body + _ws(rng)
    if rng.random() < 0.03:
        body = "﻿" + body
    if rng.random() < 0.05:
        body = rng.choice(["", "   ", "\t\r", "5", "[]", "null", "{}", "{\"text_tokens\": 5} x",
                           "{\"text_tokens\": 5,}", "{'text_tokens': 5}"])
    return body


def canonical_record(rng: random.Random) -> str:
    """write_trace's layout (the ingest fast path), with boundary values."""
    def num():
        return rng.choice([str(rng.randint(0, 3000)), "0", "00", "05", "999999999", "1000000000",
                           "2147483647", "-1", "1.0", str(rng.randint(0, 10 ** 12))])
    s = '{"text_tokens":' + (num() if rng.random() < 0.3 else str(rng.randint(0, 2000)))
    if rng.random() < 0.9:
        s += ',"image_subseqs":[' + ",".join(num() if rng.random() < 0.2 else str(v)
                                              for v in _int_list(rng)) + "]"
    if rng.random() < 0.4:
        s += ',"audio_subseqs":[' + ",".join(str(v) for v in _int_list(rng)) + "]"
    return s + "}"


def mutate(rng: random.Random, line: bytes) -> bytes:
    b = bytearray(line)
    for _ in range(rng.randint(1, 3)):
        op = rng.random()
        pos = rng.randint(0, len(b))
        if op < 0.4 and b:
            del b[min(pos, len(b) - 1)]
        elif op < 0.8:
            b.insert(pos, rng.choice(b'{}[],:"\\ 0123456789-.eE\x00\x1f\x7f\xc3\xa9\xff\xed\xa0\x80tfn'))
        elif b:
            b[min(pos, len(b) - 1)] = rng.randrange(256)
    return bytes(b).replace(b"\n", b" ")


def random_lines(seed: int, n: int) -> list:
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        line = (canonical_record(rng) if rng.random() < 0.3 else random_record(rng)).encode("utf-8")
        if rng.random() < 0.2:
            line = mutate(rng, line)
        out.append(line)
    return out


def write_trace(batch) -> bytes:
    from paper_2408_04275_b200.workload import write_trace as wt
    return wt(batch)


def synth_trace(n: int, seed: int = 1) -> bytes:
    from paper_2408_04275_b200.workload import synth_stream
    return write_trace(synth_stream(n, seed=seed))
