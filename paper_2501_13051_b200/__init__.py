"""fvlog-b200: B200-native column-oriented Datalog runtime (FVlog, arXiv 2501.13051).

The product is libfvlog.so (hand-written sm_100a CUDA + host C++ behind the C
ABI in include/fvlog.h). This package is its Python host binding:
  colog     - mirror of the reference's relation/operator API
  engine    - program / plan / fixpoint driver API
  workloads - deterministic synthetic inputs (TC, SG, CSPA, LUBM)
"""
import os

PACKAGE_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PACKAGE_DIR, "libfvlog.so")
CLI_PATH = os.path.join(PACKAGE_DIR, "fvlog")
