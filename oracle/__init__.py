"""CPU oracle for the Hydro eddy hot path.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2403_14902_b200``) never imports it and shares no code with it.
"""
from .hydro_oracle import *  # noqa: F401,F403
