"""B200-native Barnes-Hut step behind the ``nbsim`` API (arxiv 2203.08966).

Modules mirror the reference package ``nbsim`` (/root/reference/pkg/src/nbsim):
``morton``, ``physics``, ``hashed``, ``flattree``, ``integrator``,
``simulation``, ``initcond``.  Compute runs in libbh.so (hand-written sm_100a
CUDA behind a C-ABI, include/bh.h); see DESIGN.md.
"""

__version__ = "0.1.0"
