"""muxsim.simengine drop-in: only the prediction-table fixture (default_table,
offline_rate_model, InterferenceParams) is on the scheduling path; the event
engine is out of scope."""
from paper_2303_13803_b200.tables import (DEFAULT_TABLE_OFFLINE_SM, DEFAULT_TABLE_ONLINE_SM,  # noqa: F401
                                          DEFAULT_TABLE_SM_PCT, InterferenceParams, SimConfig,
                                          default_table, ground_truth_step, offline_rate_model)
