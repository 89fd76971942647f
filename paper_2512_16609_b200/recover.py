"""Scene radiance recovery and post-processing (placeholder constants)."""

DEFAULT_GAMMA = 1.2
