"""muxsim.scheduler drop-in: re-exports paper_2303_13803_b200.scheduler (GPU path)."""
from paper_2303_13803_b200.scheduler import *  # noqa: F401,F403
from paper_2303_13803_b200 import scheduler as _m

globals().update({k: getattr(_m, k) for k in dir(_m) if not k.startswith("__")})
