"""B200-native one-symbol-per-frame transducer decoding (arXiv 2211.00484).

The product is the CUDA library ``librnntg.so`` (C ABI: include/rnntg.h).
This package is a thin host-side mirror of the reference's decoder API
(rnnt-kit: ``greedy_search_batch``, ``beam_search``, ``fsa_beam_search`` +
``lattice_to_best_seq``) over that ABI, used by the tests and bench.py.
There is no CPU fallback: importing :mod:`paper_2211_00484_b200.api` loads
the in-tree library or raises.
"""

from .api import (  # noqa: F401
    BeamParams,
    Decoder,
    FsaParams,
    Graph,
    ModelWeights,
    RnntgError,
    lib_path,
)

__all__ = ["BeamParams", "Decoder", "FsaParams", "Graph", "ModelWeights", "RnntgError", "lib_path"]
