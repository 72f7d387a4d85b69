"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no alias tables, no
partitioning, no SGD): only graph/pool generators with the shapes of the
paper's workloads (tab:datasets) and the link-prediction split of
the evaluation protocol."""
from .graphs import chung_lu, dcsbm, edge_pool, linkpred_split, uniform_pool, CONFIGS  # noqa: F401
