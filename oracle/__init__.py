"""TEST INFRASTRUCTURE ONLY: the serial C oracle (gv_oracle.c) and its ctypes
wrapper (oracle.py). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package."""
