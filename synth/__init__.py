"""Seeded synthetic inputs shared by the oracle tests, smoke() and bench.py.

This package holds NONE of the method's arithmetic (no aggregation, no
partitioning, no layer math).  It only draws graphs, features, labels, train
masks and initial weights from seeded generators, with the shapes and value
distributions of the paper's workloads (Table 3).  The recipe
is stated in DESIGN.md section "Input recipe".
"""
from .graphs import CONFIGS, Graph, ModelCfg, gen_graph, glorot_params, model_for, param_count

__all__ = ["CONFIGS", "Graph", "ModelCfg", "gen_graph", "glorot_params", "model_for", "param_count"]
