"""libnfhmm: B200-native (sm_100a) VB inference for the Bayesian N-FHMM (arXiv 1206.6468).

The compute path is the C-ABI library lib/libnfhmm.so (include/nfhmm.h); `nfhmm` is its thin
ctypes binding; `synth` generates the seeded synthetic inputs of BASELINE.json's configs.
"""
__all__ = ["nfhmm", "synth"]
