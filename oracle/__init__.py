"""Test infrastructure: CPU oracles for the SolveBak sweep (see bak_oracle.py).
Never imported by the shipped package."""
