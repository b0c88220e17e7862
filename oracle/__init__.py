"""ORACLE — test infrastructure only.

CPU checkers for the GPU hot path; never imported by the product package.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
``--impl reference`` legs may load anything from here.

  ref()   the UNMODIFIED reference planner compiled from /root/reference by
          oracle/Makefile into oracle/_ref/libmmplan_ref.so (prefix mmref_).
  port()  the plain-C restatement in oracle/port/ (prefix mmport_), pinned
          against ref() and the reference's golden vectors by
          tests/test_oracle_port.py.
"""
from __future__ import annotations

import os
import subprocess

from paper_2408_04275_b200 import _capi
from paper_2408_04275_b200.api import Planner

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmmplan_ref.so")
PORT_SO = os.path.join(HERE, "_build", "libmmplan_port.so")
REF_SOURCES = "/root/reference/proj/core/src"


def build(ref: bool = True) -> None:
    """Compile the port (always) and the reference (when its sources exist),
    and the reference's own tests linked against the GPU shim
    (oracle/refcheck, needs the product library built first)."""
    targets = ["port"]
    if ref and os.path.isdir(REF_SOURCES):
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", "-C", HERE, *targets], check=True)
    if ref and os.path.isdir(REF_SOURCES):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "refcheck")], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> Planner:
    return Planner(_capi.Library(REF_SO, "mmref_"))


def port() -> Planner:
    return Planner(_capi.Library(PORT_SO, "mmport_"))


def best() -> tuple[Planner, str]:
    """The strongest oracle present: the compiled reference, else the port."""
    if ref_available():
        return ref(), "reference"
    return port(), "port"
