"""Build an experiment variant of libmuxflow.so with extra nvcc flags into
tools/_variants/NAME.so (loaded with MUX_TUNING=1 MUX_LIB_VARIANT=NAME):

    python tools/build_variant.py tie7 -DMUX_TIE_MAX=7
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_13803_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
vdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_variants")
print(B.build(extra=flags, out=os.path.join(vdir, name + ".so"), objdir=os.path.join(vdir, name + "_obj")))
