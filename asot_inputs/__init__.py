"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic)."""
from .synth import (AsotInputs, CONFIGS, EPS, anchor_sqdist_scale, make_inputs,
                    normalized_sqeuclid_cost, random_pairs)

__all__ = ["AsotInputs", "CONFIGS", "EPS", "anchor_sqdist_scale", "make_inputs",
           "normalized_sqeuclid_cost", "random_pairs"]
