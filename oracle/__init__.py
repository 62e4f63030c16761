"""fp64 CPU oracle (TEST INFRASTRUCTURE ONLY -- see oracle.py / oracle.c headers)."""
