"""Test-only CPU oracle (see lrqk_oracle.py).  Never imported by the product."""
