"""B200-native batched PCGRL env step (arXiv 2408.12525)."""
