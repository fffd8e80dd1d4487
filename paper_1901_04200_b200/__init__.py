"""B200-native two-pass ∇G engine for arXiv 1901.04200."""
