"""B200-native PLAS sort hot path (arXiv 2312.13299)."""
