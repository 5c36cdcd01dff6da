"""muxsim.predictor drop-in: re-exports paper_2303_13803_b200.predictor (GPU path)."""
from paper_2303_13803_b200.predictor import *  # noqa: F401,F403
from paper_2303_13803_b200 import predictor as _m

globals().update({k: getattr(_m, k) for k in dir(_m) if not k.startswith("__")})
