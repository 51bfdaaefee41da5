"""fmm-b200: B200-native near field (P2P + M2L) of the balanced adaptive 2D FMM (arXiv 1311.1006)."""
