"""Seeded synthetic inputs (meshes, initial states) shared by tests and bench.py.

Holds none of the DG method's arithmetic: the oracle (oracle/) and the CUDA
library (paper_1710_03887_b200/) each compute geometry, trace maps, operators,
fluxes and updates on their own from these arrays.  Recipes: SURVEY §8(c)
A5-A17 and §8(d), restated in DESIGN.md.
"""
