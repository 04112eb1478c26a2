"""Order-independent named RNG sub-streams (semantics of rrfp/rng.py:19-36).

Host-only: every random table the device consumes is drawn here, so the
device never re-implements PCG64.
"""

from __future__ import annotations

import hashlib

import numpy as np


def substream(root_seed: int, *labels) -> np.random.Generator:
    h = hashlib.blake2b(str(int(root_seed)).encode(), digest_size=16)
    for lab in labels:
        h.update(b"/%s" % str(lab).encode())
    return np.random.Generator(np.random.PCG64(int.from_bytes(h.digest(), "big")))
