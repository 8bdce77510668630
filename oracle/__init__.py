"""CPU oracle for arXiv 2005.07068 (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2005_07068_b200`` never imports it, and it never imports the product package.
"""
from .oracle import *  # noqa: F401,F403
