"""Seeded, id-addressable synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no predicate, crop, classifier,
rank or fold logic).  It only draws the inputs: detection tuples, the frame
pool, classifier weights/biases and predicate parameters.  Its hash is a
different function from the method's HASH predicate.
"""
from .workload import *  # noqa: F401,F403
