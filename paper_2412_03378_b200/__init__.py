"""B200-native analytic-transmittance Gaussian rasterizer (arXiv 2412.03378)."""
