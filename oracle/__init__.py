"""CPU parity oracle for the iFIM hot path -- TEST INFRASTRUCTURE ONLY.

A C restatement (eik_oracle.c) of the reference `eikonal` package's iFIM
engine (E/ifim.py, E/_kernels.py, E/local_solver.py, E/oracle.py), loaded
through ctypes by ``oracle.cpu``.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may import this package; the product package
paper_2106_15869_b200 never does.

Parity pins: tests/golden/*.npz, generated from the live reference by
tests/golden/make_golden.py (2D), and from a 3D generalisation of E/ifim.py
that calls the reference's own update_3d_uniform (3D).
"""
