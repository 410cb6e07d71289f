"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no attention, no softmax, no
indexing into the paged layout, no block allocation).  It only produces:

* batch *shapes*: per-request cached length c_i, new-token count n_i,
  online/offline tag and shared-prefix group (``configs``),
* token *values*: a counter-based generator that yields the same bf16 bits on
  CPU and CUDA for any (seed, tensor, content id, position, head, dim)
  coordinate (``values``), so the oracle can regenerate exactly the pieces it
  checks while the GPU path generates multi-GB KV histories in place.

The recipe (shapes, distributions, seeds) is written out in DESIGN.md §Inputs.
"""
from .configs import BatchSpec, Request, make_config, CONFIG_NAMES  # noqa: F401
from .values import q_values, kv_values, content_id  # noqa: F401
