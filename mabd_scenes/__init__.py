"""Seeded synthetic scene generators shared by the oracle and the CUDA path.

This package holds INPUTS only (geometry, masses, joint material points, initial
state). It contains none of the method's arithmetic (no polar decomposition,
no Hessians, no constraint solves), so that ``oracle/`` and the CUDA path can
both consume it without sharing any computation (task rule ③).
"""
from .generators import (  # noqa: F401
    Scene,
    make_scene,
    cfg1_chain8,
    cfg2_batched_chains,
    cfg3_long_chain,
    cfg4_binary_tree,
    cfg5_net,
    free_body,
    pendulum,
    two_body_ball,
    random_chain,
    random_tree,
    small_net,
    ring,
    box_mbar,
    CONFIG_NAMES,
)
