"""TEST INFRASTRUCTURE ONLY.

Checkers for the B200 hot path: ``oracle.ref`` drives the unmodified reference
library (oracle/_ref/librcs_ref.so, built by oracle/Makefile from
/root/reference/proj/src) and ``oracle.port`` drives our plain-C restatement
(oracle/port/rcs_port.c).  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline legs may import this package; the product package
``paper_2406_18889_b200`` never does.
"""
