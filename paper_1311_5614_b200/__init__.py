"""B200-native implicit immersed-boundary MG-FGMRES solver (arXiv 1311.5614 hot path)."""
