"""Host-side perfect-gas algebra used at setup time (initial-condition
projection, case definitions).  The per-quadrature-point versions used on
the hot path live in csrc/mhdg_math.cuh.

Same formulas as the reference's GasModel (gas.py:80-202) and ViscousParams
(gas.py:48-77) so that projected fields are bit-identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NonAdmissibleEntropyState, NonAdmissibleState


def branch_abs(x):
    return np.where(np.real(x) >= 0, x, -x)


@dataclass(frozen=True)
class ViscousParams:
    reynolds: float
    mach: float
    prandtl: float = 0.72
    mu: float = 1.0

    def shear_coefficient(self):
        return self.mu / self.reynolds

    def heat_coefficient(self, gamma):
        return self.mu / (self.reynolds * (gamma - 1) * self.mach ** 2 * self.prandtl)

    def penalty_diagonal(self, gamma, d):
        diag = np.empty(d + 2)
        diag[0] = 0.0
        diag[1:-1] = self.shear_coefficient()
        diag[-1] = self.heat_coefficient(gamma)
        return diag


@dataclass(frozen=True)
class GasModel:
    gamma: float = 1.4

    @staticmethod
    def split(u):
        return u[..., 0], u[..., 1:-1], u[..., -1]

    def primitive(self, u):
        rho, mom, rho_e = self.split(u)
        vel = mom / rho[..., None]
        p = (self.gamma - 1) * (rho_e - 0.5 * np.sum(mom * vel, axis=-1))
        return rho, vel, p

    def conservative(self, rho, vel, pressure):
        rho, vel, pressure = np.asarray(rho), np.asarray(vel), np.asarray(pressure)
        u = np.empty(vel.shape[:-1] + (vel.shape[-1] + 2,),
                     dtype=np.result_type(rho, vel, pressure, float))
        u[..., 0] = rho
        u[..., 1:-1] = rho[..., None] * vel
        u[..., -1] = pressure / (self.gamma - 1) + 0.5 * rho * np.sum(vel * vel, axis=-1)
        return u

    def pressure(self, u):
        return self.primitive(u)[2]

    def sound_speed(self, u):
        rho, _, p = self.primitive(u)
        return np.sqrt(self.gamma * p / rho)

    def check_admissible(self, u, where=""):
        rho, _, p = self.primitive(u)
        if not (np.all(np.real(rho) > 0) and np.all(np.real(p) > 0)):
            raise NonAdmissibleState("non-positive density or pressure", where=where)

    def specific_entropy(self, u):
        rho, _, p = self.primitive(u)
        return np.log(p) - self.gamma * np.log(rho)

    def entropy_density(self, u):
        return -u[..., 0] * self.specific_entropy(u) / (self.gamma - 1)

    def entropy_vars(self, u):
        rho, vel, p = self.primitive(u)
        s = np.log(p) - self.gamma * np.log(rho)
        beta = rho / p
        v = np.empty_like(u)
        v[..., 0] = (self.gamma - s) / (self.gamma - 1) - 0.5 * beta * np.sum(vel * vel, axis=-1)
        v[..., 1:-1] = beta[..., None] * vel
        v[..., -1] = -beta
        return v

    def from_entropy(self, v, where=""):
        beta = -v[..., -1]
        if not np.all(np.real(beta) > 0):
            raise NonAdmissibleEntropyState("non-positive inverse temperature", where=where)
        vel = v[..., 1:-1] / beta[..., None]
        s = self.gamma - (self.gamma - 1) * (v[..., 0] + 0.5 * beta * np.sum(vel * vel, axis=-1))
        rho = np.exp(-(s + np.log(beta)) / (self.gamma - 1))
        return self.conservative(rho, vel, rho / beta)
