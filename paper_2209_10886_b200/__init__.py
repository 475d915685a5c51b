"""B200-native hot path of the block Jacobi sweeping preconditioner (arXiv 2209.10886)."""
