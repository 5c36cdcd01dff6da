"""Drop-in `muxsim` entry points backed by the B200 implementation.

Put `pkg/src` on sys.path (as the reference's own package layout does,
/root/reference/pkg/pyproject.toml) and `from muxsim import schedule,
predict, max_weight_matching` resolves to the GPU path in
`paper_2303_13803_b200`.  Only the scheduling-round hot path is provided
(SURVEY.md §8); the simulator, CLI, trace generator and health/throttle
models of the reference are out of scope.
"""

import os as _os
import sys as _sys

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))))
if _ROOT not in _sys.path:
    _sys.path.insert(0, _ROOT)

from paper_2303_13803_b200 import *  # noqa: F401,F403,E402
from paper_2303_13803_b200 import __all__  # noqa: F401,E402
