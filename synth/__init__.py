"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

Holds no arithmetic of the method; see DESIGN.md "Input recipe"."""
from .splitmix import splitmix64, uniform01, uniform, random_permutation  # noqa: F401
from .mesh import Mesh, kuhn_mesh, config_mesh, cfd_state, cfd_dt, CONFIGS  # noqa: F401
from .graphs import (random_multigraph, path_graph, cycle_graph, fig_mot, fig_mot_alt, two_triangle,  # noqa: F401
                     int_vector, rmat, stencil2d_spmv)
