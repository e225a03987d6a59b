"""B200-native (sm_100a) LeMo contextual-token-sparsity hot path.

Drop-in for the reference ``sparsetune`` package's hot path (per-layer
token-elimination hook, pattern predictor, threshold selection and the
permutation-free sparse forward/backward of a LoRA fine-tuning step), with
every compute op implemented as a hand-written CUDA kernel in liblemo.so.
"""

__version__ = "0.1.0"
