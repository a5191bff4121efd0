"""Solver parameters (reference `pkg/src/batchsim/physics.py:54-92`)."""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class SimParams:
    dt: float = 1.0 / 120.0
    gravity: tuple = (0.0, 0.0, -9.81)
    position_iterations: int = 8
    velocity_iterations: int = 1
    max_bias: float = 0.2               # contact bias velocity = max_bias * depth / dt
    restitution: float = 0.0
    static_friction: float = 1.0
    dynamic_friction: float = 1.0
    bounce_threshold: float = 0.2       # m/s
    rest_offset: float = 0.0
    friction_offset_threshold: float = 0.04
    solver_offset_slop: float = 0.0
    friction_correlation_distance: float = 0.025
    max_force: float = 1.0e6
    linear_damping: float = 0.0
    angular_damping: float = 0.0
    max_linear_velocity: float = 1.0e3
    max_angular_velocity: float = 100.0

    def validate(self):
        """Raise ValueError on an unusable configuration (physics.py:75-92)."""
        if not self.dt > 0:
            raise ValueError("dt must be positive")
        if self.position_iterations < 1:
            raise ValueError("position_iterations must be >= 1")
        if self.velocity_iterations < 0:
            raise ValueError("velocity_iterations must be >= 0")
        if not 0.0 <= self.restitution <= 1.0:
            raise ValueError("restitution must be in [0, 1]")
        vals = (self.max_bias, self.static_friction, self.dynamic_friction,
                self.bounce_threshold, self.rest_offset, self.max_force,
                self.linear_damping, self.angular_damping,
                self.max_linear_velocity, self.max_angular_velocity, *self.gravity)
        if not all(math.isfinite(float(v)) for v in vals):
            raise ValueError("params must be finite")
        if self.max_linear_velocity <= 0 or self.max_angular_velocity <= 0:
            raise ValueError("velocity limits must be positive")
        return self
