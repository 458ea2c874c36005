"""Test-infrastructure CPU oracle (see camarray_oracle.py header).

Never imported by the product package `paper_1910_03517_b200`."""
