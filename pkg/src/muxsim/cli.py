"""muxsim.cli drop-in: the hot-path subcommands (schedule, match, predict) on
the GPU round; the simulator subcommands are out of scope."""
from paper_2303_13803_b200.cli import *  # noqa: F401,F403
from paper_2303_13803_b200.cli import main  # noqa: F401
