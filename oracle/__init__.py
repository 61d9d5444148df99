"""fp64 CPU oracle for the arXiv 1707.02018 hot path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference
leg) may import this package.  It shares no code with paper_1707_02018_b200/.
"""
