"""TEST INFRASTRUCTURE ONLY: CPU checkers for the NGF + curvature path (see oracle.py)."""
