"""B200-native batched linear elliptical slice sampling (arXiv 2407.10449)."""
