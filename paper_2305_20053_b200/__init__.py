"""B200-native SAA risk / control-gradient engine for MR-DINO surrogates
(arxiv 2305.20053).  Host API mirrors the reference package's hot-path
surface (ouukit/__init__.py:5-22); the compute runs in libsaadino.so
(hand-written sm_100a CUDA, include/saadino.h)."""

from .api import (Decoder, NetworkSpec, OptResult, ReducedTrackingForm, RiskSpec, SAAProblem, SurrogateErrors,
                  SurrogateEvaluator, SurrogateModel, build_tracking_form, evaluate_errors, init_model,
                  mc_cvar, mc_var, minimize, saa_objective, splus, splus_d1)
from .engine import Engine, EvalResult
from . import fileio, workloads
from .training import TrainConfig, TrainingDivergedError, loss_and_grad, train

__version__ = "0.1.0"

__all__ = ["TrainConfig", "TrainingDivergedError", "loss_and_grad", "train", "SurrogateErrors", "evaluate_errors", "Decoder", "Engine", "EvalResult", "NetworkSpec", "OptResult", "ReducedTrackingForm", "RiskSpec", "minimize",
           "SAAProblem", "SurrogateEvaluator", "SurrogateModel", "build_tracking_form", "init_model",
           "mc_cvar", "mc_var", "saa_objective", "splus", "splus_d1", "fileio", "workloads"]
