"""B200-native latent-map optimisation step (LatentAM, arxiv 2602.12314).

Hand-written sm_100a CUDA kernels behind the C-ABI of include/latmap_b200.h
(liblatmap_b200.so); see DESIGN.md. Importing the package does not need a GPU;
every compute call does, and fails loudly without one (no CPU fallback).
"""
from ._capi import LIB_PATH, InvalidArgument, LatmapError, StaleCache, lib  # noqa: F401

__all__ = ["lib", "LIB_PATH", "LatmapError", "InvalidArgument", "StaleCache"]
