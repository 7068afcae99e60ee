"""CPU oracles — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the
CPU baseline. The product path (paper_1810_03988_b200) never imports it.

Two oracles share one numpy-level interface (class Oracle):
  kind="ref": the reference itself, compiled from /root/reference headers
              (oracle/_ref/liblorbref.so, built by oracle/Makefile);
  kind="orc": the plain-C restatement oracle/lorb_oracle.c
              (oracle/_build/liborc.so), pinned to "ref" by tests/golden.
"""
from .oracle import Oracle, build, ref_available, orc_available  # noqa: F401
