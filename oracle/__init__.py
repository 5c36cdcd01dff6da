"""CPU oracle for the MuxFlow scheduling round -- TEST INFRASTRUCTURE ONLY.

This package is a CPU restatement of the reference's hot path
(`/root/reference/pkg/src/muxsim/predictor.py`, `matching.py`,
`scheduler.py`).  It exists so that the CUDA product path can be checked
against it.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it, and only as the
checker or the CPU baseline -- never as the thing measured or shipped.
The product package `paper_2303_13803_b200` never imports this package.

Parity status: PINNED.  `tests/test_oracle_golden.py` checks every function
here against golden vectors produced by running the reference itself
(`tests/golden/make_golden.py`, committed with its outputs).  The MLP
predictor oracle (`oracle/mlp_ref.py`) has no reference counterpart: parity
unpinned for that plugin only.
"""
