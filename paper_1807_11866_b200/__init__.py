"""B200-native batched online solver for the velocity-only reduced Navier–Stokes method (arXiv 1807.11866)."""
