"""B200-native evaluator for phi = sum_k c_k prod_t A_{k_t} (arXiv 2202.04140).

Drop-in for the evaluation path of the reference package ``acedag``
(/root/reference/pkg/src/acedag/__init__.py:4-64): the same names for the
basis specification, the DAG and the evaluators, backed by hand-written
sm_100a CUDA kernels behind the C ABI in include/acedag_b200.h.  The batched
production API is :class:`SitePlan`.
"""

from .indexsets import (DegreeSpec, Group, canonical, element_degree, format_elements,
                        one_particle_indices, parse_elements, satisfies_constraints, tuple_degree)
from .graph import (EvalGraph, GraphFormatError, GraphNode, UnsupportedVersionError, as_eval_graph,
                    build_graph, deserialize_graph, graph_from_parents, read_graph, seed_graph,
                    serialize_graph, write_graph)
from .evaluator import (InvarianceReport, SitePlan, evaluate_graph, evaluate_model, invariance_check,
                        invert_particles, launch_count, naive_eval, naive_products, one_particle, pool,
                        pool_batched,
                        pool_positions, random_particles, read_coefficients, read_particles,
                        rotate_particles, write_coefficients, write_particles)

__version__ = "0.1.0"
