"""TEST INFRASTRUCTURE -- the CHECKERS, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg (cpu_baseline,
--impl reference) may import this package. It wraps:
  * oracle/_ref/libperiwave_ref.so -- the UNMODIFIED reference library compiled from
    /root/reference/proj/src with own GSL/FFTW shims (oracle/Makefile);
  * oracle/_build/libperiwave_port.so -- the plain-C restatement (oracle/port/).
Parity pinning: the port and the shims are checked against the reference's own
known answers (proj/tests/test_kernels.cpp:28-48 etc.) and against _ref outputs in
tests/test_oracle_pins.py; golden fixtures in tests/golden/ come from _ref.
"""
