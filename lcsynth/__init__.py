"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module only *synthesises* worlds (cameras, keyframes, features, map points,
loop events). It holds none of the method's arithmetic: it never calls `oracle/`
or the CUDA library, and neither of those imports it. Random numbers the method
would draw do not exist (the method is deterministic).
"""
from .world import CAMERAS, CONFIGS, World, make_world  # noqa: F401
from .posegraph import GRAPHS, PoseGraph, make_pose_graph  # noqa: F401
