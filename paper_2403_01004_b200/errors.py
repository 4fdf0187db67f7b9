"""Exceptions of the path, mirroring the SPEC's error contracts.

  InvalidGridError (ValueError)  mesh.py:32-33 (re-exported from ``mesh``)
  IndefiniteOperatorError        PCG breakdown p^T A p <= 0 / non-positive Jacobi
                                 diagonal
  DivergenceError                NaN in the PCG residual
  BlowUpError(stage)             non-finite STS stage, naming the stage
  CycleCapError(report)          max_cycles exceeded, carrying the partial report
                                 
  DomainError (ValueError)       non-positive T0 for aligned conduction
"""
from __future__ import annotations


class ParacycleError(RuntimeError):
    pass


class NativeLibraryMissing(ImportError):
    pass


class DeviceError(ParacycleError):
    pass


class CommError(ParacycleError):
    pass


class IndefiniteOperatorError(ArithmeticError):
    pass


class DivergenceError(ArithmeticError):
    pass


class BlowUpError(FloatingPointError):
    def __init__(self, stage: int, msg: str = ""):
        super().__init__(msg or f"non-finite value at stage {stage}")
        self.stage = stage


class CycleCapError(RuntimeError):
    def __init__(self, msg: str, report=None):
        super().__init__(msg)
        self.report = report


class NotConvergedError(ArithmeticError):
    def __init__(self, msg: str, report=None):
        super().__init__(msg)
        self.report = report


class DomainError(ValueError):
    pass
