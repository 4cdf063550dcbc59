"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no fit, no projection, no
search): it only draws database vectors, query vectors, the learning-row
sample and the uniform draws that k-means++ consumes.  Both sides (oracle/
and the product path) import it; neither imports the other.
"""
from .gen import (CONFIGS, Config, get_config, database, database_rows, queries,
                  learn_rows, kmeanspp_draws, full_dtype_np)

__all__ = ["CONFIGS", "Config", "get_config", "database", "database_rows", "queries",
           "learn_rows", "kmeanspp_draws", "full_dtype_np"]
