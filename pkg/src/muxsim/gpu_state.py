"""muxsim.gpu_state drop-in: only HealthState is on the scheduling path."""
from paper_2303_13803_b200.core import HealthState  # noqa: F401
