"""B200-native sliced tensor-network contraction executor (arXiv 2002.01935 hot path)."""
