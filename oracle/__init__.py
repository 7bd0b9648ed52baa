"""TEST INFRASTRUCTURE — ORACLE, NOT PRODUCT.

CPU checkers for the fvlog CUDA path. Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / reference legs may import this package, and
only as the checker or the timed CPU baseline — never as the thing measured
on the GPU path. The product (paper_2501_13051_b200) never imports it.

  oracle.bind.Oracle     ctypes over oracle/liboracle.so, the plain-C
                         restatement of the reference algorithms
                         (oracle/colog_oracle.c)
  oracle.bind.Reference  ctypes over oracle/_ref/libcolog_ref.so, the
                         UNMODIFIED reference compiled by oracle/Makefile
                         (present only where /root/reference was available)
  oracle.naive           pure-Python naive least-model evaluator restating
                         P/src/oracle.cpp (small inputs only)
"""
