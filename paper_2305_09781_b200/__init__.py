"""spectree-b200: B200-native (sm_100a) token-tree verification for SpecInfer.

Drop-in for the reference's token-tree / tree-attention / verify path
(reference: proj/include/spectree/*.hpp). Layers:

* ``libspectree_b200.so`` — hand-written CUDA kernels (K1 tree attention,
  K2 KV append/compaction, K3 greedy verify, K4 multi-step speculative
  sampling) and the host C++ token-tree library, behind the C-ABI
  ``include/spectree_capi.h``;
* ``paper_2305_09781_b200._capi`` — ctypes binding of that C-ABI over torch
  device tensors (torch = memory/streams plumbing only);
* ``paper_2305_09781_b200.tree`` — the reference's Python-facing tree API
  (``TokenTree.merge_sequences``, ``verify``) over the C++ host library.
"""
from ._capi import SpectreeError, lib  # noqa: F401

__all__ = ["SpectreeError", "lib"]
