"""B200-native nonlocal stiffness/load assembly (arXiv 2101.08825 hot path).

Drop-in for the reference package's assembly path (mollifem/__init__.py:3-13):
the same `build_mesh`, `FESpace`, `KernelParams`, `AssemblyConfig`,
`assemble`, `assemble_rhs`, `neighbor_sets`, `SparseMatrix` names and
contracts, with every kernel on the path running as hand-written sm_100a
CUDA through the C-ABI in include/mollifem_b200.h.
"""

from .assembly import (AssemblyConfig, NeighborSets, SparseMatrix,
                       aprx_max_dist, aprx_min_dist, assemble, assemble_rhs,
                       neighbor_sets,
                       pattern_halfwidth)
from .fe_space import (FESpace, eval_basis, eval_shape_functions,
                       interpolate, l2_error, lifting)
from .kernel import (KernelParams, gamma_eps, mollifier, scaling_c_delta,
                     scaling_c_delta_eps, xi)
from .mesh import (BoundingBox, DelaunayMesh, Mesh, PartitionMap,
                   build_delaunay_mesh, build_mesh, partition_geometric,
                   refine)
from .solver import SolveReport, solve
from .quadrature import (QuadratureRule, dunavant6, dunavant7, strang3,
                         gauss_legendre_1d,
                         gauss_lobatto_1d, map_to_physical, rule_for_kind,
                         tensor_product)

__version__ = "0.1.0"

__all__ = [
    "AssemblyConfig", "BoundingBox", "DelaunayMesh", "FESpace",
    "KernelParams", "Mesh",
    "NeighborSets", "PartitionMap", "QuadratureRule", "SparseMatrix",
    "aprx_max_dist", "aprx_min_dist", "assemble", "assemble_rhs",
    "build_delaunay_mesh", "build_mesh", "dunavant6", "dunavant7", "strang3",
    "eval_basis", "eval_shape_functions", "gamma_eps", "gauss_legendre_1d",
    "gauss_lobatto_1d", "interpolate", "l2_error", "lifting",
    "map_to_physical", "mollifier", "neighbor_sets", "partition_geometric",
    "pattern_halfwidth", "refine", "rule_for_kind", "scaling_c_delta",
    "scaling_c_delta_eps", "solve", "SolveReport", "tensor_product", "xi",
]
