"""Dark channel, atmospheric light, transmission and guided refinement (placeholder constants)."""

DEFAULT_PATCH_RADIUS = 7
DEFAULT_TOP_FRACTION = 0.001
DEFAULT_ALPHA = 0.8
DEFAULT_OMEGA = 0.5
DEFAULT_T_MIN = 0.05
DEFAULT_GUIDED_RADIUS = 40
DEFAULT_GUIDED_EPS = 1e-3
AIRLIGHT_FLOOR = 1e-6
