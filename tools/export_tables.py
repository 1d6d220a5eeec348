#!/usr/bin/env python
"""Write oracle/tables/kfvm_table_d{dim}_r{R}.npz: the canonical reconstruction
tables (binary128 precompute of libkfvm_b200.so, rounded once to FP64) as
plain arrays with their FNV-1a hash.

The CPU reference arm of bench.py loads these files through
oracle/table_file.py, so timing the reference never maps the product
library; tests/test_table_file.py checks that the files equal the live
precompute byte for byte.  Re-run after any change to the precompute."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2401_16543_b200 as K  # noqa: E402
from oracle.table_file import FIELDS, table_arrays  # noqa: E402


def main():
    out = os.path.join(ROOT, "oracle", "tables")
    os.makedirs(out, exist_ok=True)
    for dim, R in ((2, 2), (2, 3), (3, 2), (3, 3)):
        rset = K.precompute(R, dim=dim)
        arr = table_arrays(rset.c_table.contents)
        assert set(arr) == set(FIELDS)
        path = os.path.join(out, f"kfvm_table_d{dim}_r{R}.npz")
        np.savez_compressed(path, **arr)
        print(f"{path}: hash {int(arr['hash'][0]):#018x}")


if __name__ == "__main__":
    main()
