"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the CUDA path.

`oracle.C` binds oracle/_build/libgx_oracle.so (the plain-C restatement in
oracle/gx_oracle.c). `oracle.REF` binds oracle/_ref/libgx_ref.so (the UNMODIFIED
reference headers compiled by oracle/Makefile) when it has been built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
may import this package. The product package (paper_2208_09151_b200) never does.
"""
from .bind import (OracleError, C, GEN, REF, ref_available, build,  # noqa: F401
                   oracle_lib_path, ref_lib_path)
