"""Import the UNMODIFIED reference simulator ``ditsim`` for boundary tests (tests only).

Order: ``baseline/_ref`` (the one offline install of the reference, `pip install --no-deps
--target baseline/_ref`, which travels to the GPU box), then the read-only source tree in this
container. Skips when neither exists."""
import importlib
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]


def ditsim():
    for p in CANDIDATES:
        if (p / "ditsim" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return importlib.import_module("ditsim")
    pytest.skip("the reference ditsim package is not installed (baseline/_ref)")
