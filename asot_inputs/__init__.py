"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic)."""
from .synth import AsotInputs, CONFIGS, EPS, make_inputs, normalized_sqeuclid_cost, random_pairs

__all__ = ["AsotInputs", "CONFIGS", "EPS", "make_inputs", "normalized_sqeuclid_cost", "random_pairs"]
