"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds the config table (BASELINE.json configs[0..4]) and the input
recipe: density field -> cone filter -> Heaviside projection -> SIMP moduli,
boundary masks, consistent nodal loads and the smooth adjoint right-hand sides.
It contains none of the hot path's arithmetic (no stiffness, no solve, no G):
both `oracle/` and the product path consume its arrays, and neither imports the
other.  See DESIGN.md "Input recipe" for the readings.
"""

from .configs import CONFIGS, Config, get_config, level_dims, n_nodes, n_dofs, n_elems
from .generate import generate, rough_vectors, element_grid_shape, node_grid_shape

__all__ = [
    "CONFIGS", "Config", "get_config", "level_dims", "n_nodes", "n_dofs", "n_elems",
    "generate", "rough_vectors", "element_grid_shape", "node_grid_shape",
]
