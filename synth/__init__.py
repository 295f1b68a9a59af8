"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no normalisation, no
aggregation, no transform, no loss): it only draws graphs, features and labels
with the shapes and structure of the paper's workloads.
Both `oracle/` and the product consume its arrays; neither imports the other.
"""
from .generate import (CONFIGS, WorkloadConfig, make_graph, make_features,
                       make_labels, make_workload, make_sbm_toy)

__all__ = ["CONFIGS", "WorkloadConfig", "make_graph", "make_features",
           "make_labels", "make_workload", "make_sbm_toy"]
