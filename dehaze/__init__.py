"""`dehaze` import name for the B200 drop-in: `import dehaze` / `from dehaze.pipeline import ...`
resolve to paper_2512_16609_b200 (so code written against the reference package runs unchanged)."""

import importlib
import sys

import paper_2512_16609_b200 as _pkg
from paper_2512_16609_b200 import *  # noqa: F401,F403
from paper_2512_16609_b200 import __all__, __getattr__, __version__  # noqa: F401

for _name in ("estimation", "imageops", "morphology", "pipeline", "recover", "synth", "benchmark", "validation",
              "estimator", "frameio"):
    sys.modules[f"{__name__}.{_name}"] = importlib.import_module(f"{_pkg.__name__}.{_name}")
