"""B200-native EXACT-MPPI rollout + exact signed-distance hot path.

The compute lives in libexm_b200.so (hand-written sm_100a CUDA behind the C ABI of
include/exm_b200.h); this package is the host-side mirror of the reference's controller API.
"""
from .api import (ComponentLimit, ControlDecision, Engine, FootprintSpec, Guidance,
                  KinematicLimits, MotionModel, MppiController, MppiParams, ObstacleSet,
                  RolloutBatch, TaskWeights)

__all__ = ["ComponentLimit", "ControlDecision", "Engine", "FootprintSpec", "Guidance",
           "KinematicLimits", "MotionModel", "MppiController", "MppiParams", "ObstacleSet",
           "RolloutBatch", "TaskWeights"]
