"""Synthetic tracking data for the benchmark and tests.

Stationary 2-D constant-velocity model: dt = 0.1,
F = [[rho_p, 0, dt, 0], [0, rho_p, 0, dt], [0, 0, rho_v, 0], [0, 0, 0, rho_v]]
with rho_p = 0.99, rho_v = 0.95; Q = q [[dt^3/3 I, dt^2/2 I], [dt^2/2 I, dt I]],
q = 1; H = [I_2 0]; R = 0.25 I_2; u = d = 0; prior mean (0, 0, 1, -1), prior
cov I.  The damping keeps the series stationary so both the FP64 (1e-9) and
FP32 (1e-4) parity gates are meaningful at T = 2^24 (the undamped model breaks
the reference's own parallel-vs-sequential agreement, SURVEY.md 7 hard part 3).

Measurements are drawn by ancestral sampling with numpy's PCG64 stream; the
state recursion runs as two first-order linear filters (scipy lfilter) so
T = 2^24 takes a few seconds.  ``time_varying=True`` writes the model per step
(the reference API is per step, lgssm.hpp:29-42); ``False`` keeps single
blocks (stride-0 broadcast).
"""
from __future__ import annotations

import numpy as np

from .api import Lgssm


def cv_matrices(dt: float = 0.1, rho_p: float = 0.99, rho_v: float = 0.95,
                q: float = 1.0, r: float = 0.25):
    F = np.array([[rho_p, 0, dt, 0], [0, rho_p, 0, dt], [0, 0, rho_v, 0],
                  [0, 0, 0, rho_v]], dtype=np.float64)
    I2 = np.eye(2)
    Q = q * np.block([[dt ** 3 / 3 * I2, dt ** 2 / 2 * I2],
                      [dt ** 2 / 2 * I2, dt * I2]])
    H = np.hstack([I2, np.zeros((2, 2))])
    R = r * I2
    m0 = np.array([0.0, 0.0, 1.0, -1.0])
    P0 = np.eye(4)
    return F, Q, H, R, m0, P0


def simulate_cv(t: int, seed: int = 0, dt: float = 0.1, rho_p: float = 0.99,
                rho_v: float = 0.95, q: float = 1.0, r: float = 0.25) -> np.ndarray:
    """Measurements y[T][2] of the damped CV model (float64)."""
    from scipy.signal import lfilter

    F, Q, H, R, m0, P0 = cv_matrices(dt, rho_p, rho_v, q, r)
    rng = np.random.Generator(np.random.PCG64(seed))
    x0 = m0 + np.linalg.cholesky(P0) @ rng.standard_normal(4)
    w = rng.standard_normal((t, 4)) @ np.linalg.cholesky(Q).T  # state noise
    # velocities: v_{k+1} = rho_v v_k + w_v   (k = 0..T-1, x_{k+1} is step k+1)
    vel = np.empty((t, 2))
    pos = np.empty((t, 2))
    for a in range(2):
        v_in = w[:, 2 + a].copy()
        v_in[0] += rho_v * x0[2 + a]
        vel[:, a] = lfilter([1.0], [1.0, -rho_v], v_in)
        # p_{k+1} = rho_p p_k + dt v_k + w_p ; v_k is the previous velocity
        v_prev = np.concatenate([[x0[2 + a]], vel[:-1, a]])
        p_in = dt * v_prev + w[:, a]
        p_in[0] += rho_p * x0[a]
        pos[:, a] = lfilter([1.0], [1.0, -rho_p], p_in)
    y = pos + rng.standard_normal((t, 2)) * np.sqrt(r)
    return y


def cv_model(t: int, seed: int = 0, dtype=np.float64, time_varying: bool = True,
             **kw) -> tuple[Lgssm, np.ndarray]:
    """(model, ys) for the damped CV tracking problem."""
    F, Q, H, R, m0, P0 = cv_matrices(**{k: v for k, v in kw.items()
                                        if k in ("dt", "rho_p", "rho_v", "q", "r")})
    ys = simulate_cv(t, seed, **kw).astype(dtype)
    u = np.zeros(4)
    d = np.zeros(2)

    def per_step(a):
        a = a.astype(dtype)
        return np.ascontiguousarray(np.broadcast_to(a, (t, *a.shape))) if time_varying else a

    m = Lgssm(f=per_step(F), u=per_step(u), q=per_step(Q), h=per_step(H),
              d=per_step(d), r=per_step(R), prior_mean=m0.astype(dtype),
              prior_cov=P0.astype(dtype), t=t)
    return m, ys
