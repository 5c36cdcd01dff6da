"""Build the oracle's C restatement (TEST INFRASTRUCTURE ONLY).

Compiles oracle/hungarian.c into oracle/build/liboracle.so with plain gcc.
Called by __graft_entry__.build() and lazily by oracle.matching_ref.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build():
    out_dir = os.path.join(HERE, "build")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "liboracle.so")
    srcs = [os.path.join(HERE, "hungarian.c")]
    if os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(s) for s in srcs):
        return out
    # -ffp-contract=off: no FMA contraction, so float64 arithmetic matches numpy
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", out + ".tmp"] + srcs + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build())
