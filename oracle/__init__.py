"""TEST INFRASTRUCTURE ONLY (see oracle/tgx_oracle.h): ctypes bindings to the
checkers. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this package; the product never does."""
