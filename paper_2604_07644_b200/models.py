"""Plant models: the contract the SQP/SLS layers linearize, plus device twins.

``Model`` mirrors the reference ABC (/root/reference/pkg/src/scanmpc/models.py:37-93):
``step``, ``jacobians``, stage/terminal constraints with Jacobians,
``disturbance`` E(x), constant quadratic ``cost_weights`` and a ``reference``.
The host-side methods here are the *specification* of each plant (numpy,
float64); the ones with a CUDA twin expose ``device_spec()`` and are
linearized on the GPU by ``gsls_linearize`` (csrc/models.cu).

Plants:

* ``DubinsCar``, ``PlanarQuadrotor``, ``NLinkPendulum`` — the reference's
  fixtures (models.py:130-448), same parameters and formulas.
* ``Quadrotor12`` — 12D rigid-body quadrotor (p, euler, v, omega; 4 rotor
  thrusts; RK4), the BASELINE cfg-B/C plant.
* ``SyntheticLegged`` — seeded stable nonlinear plant of legged-robot shape
  (61D/12u quadruped, 75D/19u humanoid; BASELINE cfg-D/E) with a torque
  box and obstacle rows on (x0, x1).

Every constraint set here has the form
``[u - u_max; u_min - u; r^2 - |x[:2] - c|^2 (per obstacle)]`` — the device
linearizer implements that one family.
"""

from __future__ import annotations

import abc
from dataclasses import dataclass, field

import numpy as np

GRAVITY = 9.81

# device model ids (csrc/models.cu)
DEV_DUBINS, DEV_PLANAR_QUAD, DEV_PENDULUM, DEV_QUAD12, DEV_SYNTH = 1, 2, 3, 4, 5


def obstacle_values(px, py, obstacles) -> np.ndarray:
    """r^2 - (px-cx)^2 - (py-cy)^2 per obstacle (models.py:20-25)."""
    return np.array([r * r - (px - cx) ** 2 - (py - cy) ** 2 for cx, cy, r in obstacles], dtype=float)


def obstacle_position_jacobian(px, py, obstacles) -> np.ndarray:
    """models.py:28-34."""
    J = np.empty((len(obstacles), 2))
    for i, (cx, cy, _r) in enumerate(obstacles):
        J[i] = (-2.0 * (px - cx), -2.0 * (py - cy))
    return J


def complex_step_jacobians(step, x, u, h: float = 1e-30):
    """Exact (to rounding) Jacobians of an analytic step map by complex steps."""
    x = np.asarray(x, float)
    u = np.asarray(u, float)
    nx, nu = x.shape[0], u.shape[0]
    A = np.empty((nx, nx))
    B = np.empty((nx, nu))
    for i in range(nx):
        xc = x.astype(complex)
        xc[i] += 1j * h
        A[:, i] = np.imag(step(xc, u.astype(complex))) / h
    for i in range(nu):
        uc = u.astype(complex)
        uc[i] += 1j * h
        B[:, i] = np.imag(step(x.astype(complex), uc)) / h
    return A, B


def rk4(fc, x, u, dt):
    k1 = fc(x, u)
    k2 = fc(x + 0.5 * dt * k1, u)
    k3 = fc(x + 0.5 * dt * k2, u)
    k4 = fc(x + dt * k3, u)
    return x + (dt / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)


class Model(abc.ABC):
    """Interface consumed by linearize / SLS (models.py:37-93)."""

    nx: int
    nu: int
    dt: float

    @abc.abstractmethod
    def step(self, x, u): ...

    @abc.abstractmethod
    def jacobians(self, x, u): ...

    @abc.abstractmethod
    def stage_constraints(self, x, u): ...

    @abc.abstractmethod
    def stage_constraint_jacobians(self, x, u): ...

    def terminal_constraints(self, x):
        return np.zeros(0)

    def terminal_constraint_jacobian(self, x):
        return np.zeros((0, self.nx))

    @abc.abstractmethod
    def disturbance(self, x): ...

    def clip_input(self, u):
        return u

    @property
    def nc(self) -> int:
        return self.stage_constraints(np.zeros(self.nx), np.zeros(self.nu)).shape[0]

    @property
    def nf(self) -> int:
        return self.terminal_constraints(np.zeros(self.nx)).shape[0]

    @abc.abstractmethod
    def cost_weights(self): ...

    @abc.abstractmethod
    def reference(self, N): ...

    def tracking_cost(self, x, u) -> float:
        Q, R, QN = self.cost_weights()
        xref, uref = self.reference(u.shape[0])
        ex, eu = x - xref, u - uref
        J = 0.5 * float(np.einsum("ki,ij,kj->", ex[:-1], Q, ex[:-1]))
        J += 0.5 * float(np.einsum("ki,ij,kj->", eu, R, eu))
        return J + 0.5 * float(ex[-1] @ QN @ ex[-1])

    # -- device twin ---------------------------------------------------------
    def device_spec(self):
        """(model_id, model parameters, constraint block) for csrc/models.cu, or None.

        The constraint block is ``[n_obs, u_min (nu), u_max (nu), (cx, cy, r) * n_obs]``.
        """
        return None


class _BoxObstacleModel(Model):
    """Shared constraint family: input box + obstacle rows on (x0, x1)."""

    def _u_bounds(self):
        raise NotImplementedError

    def _obstacles(self):
        return tuple(getattr(self, "obstacles", ()))

    def stage_constraints(self, x, u):
        lo, hi = self._u_bounds()
        return np.concatenate([u - hi, lo - u, obstacle_values(x[0], x[1], self._obstacles())])

    def stage_constraint_jacobians(self, x, u):
        n_obs = len(self._obstacles())
        C = np.zeros((2 * self.nu + n_obs, self.nx))
        C[2 * self.nu:, :2] = obstacle_position_jacobian(x[0], x[1], self._obstacles())
        D = np.vstack([np.eye(self.nu), -np.eye(self.nu), np.zeros((n_obs, self.nu))])
        return C, D

    def terminal_constraints(self, x):
        return obstacle_values(x[0], x[1], self._obstacles())

    def terminal_constraint_jacobian(self, x):
        CN = np.zeros((len(self._obstacles()), self.nx))
        CN[:, :2] = obstacle_position_jacobian(x[0], x[1], self._obstacles())
        return CN

    def clip_input(self, u):
        lo, hi = self._u_bounds()
        return np.clip(u, lo, hi)

    def _constraint_params(self):
        lo, hi = self._u_bounds()
        obs = np.asarray(self._obstacles(), float).reshape(-1, 3)
        return np.concatenate([[len(obs)], np.broadcast_to(lo, (self.nu,)),
                               np.broadcast_to(hi, (self.nu,)), obs.ravel()])


@dataclass(frozen=True)
class DubinsCar(_BoxObstacleModel):
    """Constant-speed Dubins car, forward Euler (models.py:130-201)."""

    v: float = 1.0
    dt: float = 0.1
    omega_max: float = 2.0
    obstacles: tuple = ()
    goal: tuple = (4.0, 0.0, 0.0)
    q_diag: tuple = (1.0, 1.0, 0.1)
    r_diag: tuple = (0.1,)
    qn_diag: tuple = (10.0, 10.0, 1.0)
    e_scale: float = 2.5e-2
    nx: int = field(default=3, init=False)
    nu: int = field(default=1, init=False)

    def step(self, x, u):
        return np.array([x[0] + self.v * np.cos(x[2]) * self.dt,
                         x[1] + self.v * np.sin(x[2]) * self.dt,
                         x[2] + u[0] * self.dt])

    def jacobians(self, x, u):
        A = np.eye(3)
        A[0, 2] = -self.v * np.sin(x[2]) * self.dt
        A[1, 2] = self.v * np.cos(x[2]) * self.dt
        return A, np.array([[0.0], [0.0], [self.dt]])

    def _u_bounds(self):
        return np.array([-self.omega_max]), np.array([self.omega_max])

    def disturbance(self, x):
        return self.e_scale * np.eye(3)

    def cost_weights(self):
        return np.diag(self.q_diag), np.diag(self.r_diag), np.diag(self.qn_diag)

    def reference(self, N):
        return np.tile(np.asarray(self.goal, float), (N + 1, 1)), np.zeros((N, 1))

    def device_spec(self):
        return DEV_DUBINS, np.array([self.v, self.dt], float), self._constraint_params()


@dataclass(frozen=True)
class PlanarQuadrotor(_BoxObstacleModel):
    """Planar quadrotor, RK4 (models.py:204-299)."""

    m: float = 2.0576
    L: float = 0.25
    J: float = 0.01
    dt: float = 0.02
    thrust_max: float = 40.0
    obstacles: tuple = ()
    goal: tuple = (3.0, 0.0, 0.0, 0.0, 0.0, 0.0)
    q_diag: tuple = (1.0, 1.0, 0.5, 0.1, 0.1, 0.05)
    r_diag: tuple = (0.05, 0.05)
    qn_diag: tuple = (20.0, 20.0, 5.0, 1.0, 1.0, 0.5)
    e_scale: float = 5e-2
    nx: int = field(default=6, init=False)
    nu: int = field(default=2, init=False)

    def f_cont(self, x, u):
        phi, vx, vy, om = x[2], x[3], x[4], x[5]
        T = u[0] + u[1]
        return np.array([vx, vy, om, -T * np.sin(phi) / self.m,
                         T * np.cos(phi) / self.m - GRAVITY, self.L * (u[1] - u[0]) / self.J])

    def step(self, x, u):
        return rk4(self.f_cont, np.asarray(x), np.asarray(u), self.dt)

    def jacobians(self, x, u):
        return complex_step_jacobians(self.step, x, u)

    def hover_thrust(self):
        return self.m * GRAVITY / 2.0

    def _u_bounds(self):
        return np.zeros(2), np.full(2, self.thrust_max)

    def disturbance(self, x):
        return self.e_scale * np.diag([0.0, 0.0, 0.0, 1.0, 1.0, 0.0])

    def cost_weights(self):
        return np.diag(self.q_diag), np.diag(self.r_diag), np.diag(self.qn_diag)

    def reference(self, N):
        return (np.tile(np.asarray(self.goal, float), (N + 1, 1)),
                np.full((N, 2), self.hover_thrust()))

    def device_spec(self):
        return DEV_PLANAR_QUAD, np.array([self.m, self.L, self.J, self.dt], float), self._constraint_params()


@dataclass(frozen=True)
class NLinkPendulum(_BoxObstacleModel):
    """Serial n-link pendulum, semi-implicit Euler (models.py:302-448)."""

    n_links: int = 2
    masses: tuple = None
    lengths: tuple = None
    dt: float = 0.01
    u_max: float = 20.0
    q_angle: float = 10.0
    q_rate: float = 1.0
    r_torque: float = 0.05
    qn_scale: float = 10.0
    e_rate: float = 0.0

    def __post_init__(self):
        n = self.n_links
        if self.masses is None:
            object.__setattr__(self, "masses", tuple(1.0 for _ in range(n)))
        if self.lengths is None:
            object.__setattr__(self, "lengths", tuple(1.0 for _ in range(n)))
        m = np.asarray(self.masses, float)
        l = np.asarray(self.lengths, float)
        lever = np.zeros((n, n))
        for k in range(n):
            lever[k, :k] = l[:k]
            lever[k, k] = 0.5 * l[k]
        object.__setattr__(self, "_kappa", np.einsum("k,ki,kj->ij", m, lever, lever))
        object.__setattr__(self, "_inertia", m * l ** 2 / 12.0)
        object.__setattr__(self, "_glever", GRAVITY * (m[:, None] * lever).sum(axis=0))
        T = np.eye(n)
        T[np.arange(n - 1), np.arange(1, n)] = -1.0
        object.__setattr__(self, "_tmap", T)

    @property
    def nx(self):
        return 2 * self.n_links

    @property
    def nu(self):
        return self.n_links

    def accel(self, x, u):
        n = self.n_links
        th, om = x[:n], x[n:]
        d = th[:, None] - th[None, :]
        M = self._kappa * np.cos(d) + np.diag(self._inertia)
        bias = (self._kappa * np.sin(d)) @ (om ** 2) + self._glever * np.sin(th)
        try:
            return np.linalg.solve(M, self._tmap @ u - bias)
        except np.linalg.LinAlgError as exc:
            raise ArithmeticError("pendulum mass matrix is singular") from exc

    def step(self, x, u):
        n = self.n_links
        om = x[n:] + self.dt * self.accel(x, u)
        return np.concatenate([x[:n] + self.dt * om, om])

    def jacobians(self, x, u):
        return complex_step_jacobians(self.step, x, u)

    def _u_bounds(self):
        return np.full(self.n_links, -self.u_max), np.full(self.n_links, self.u_max)

    def _obstacles(self):
        return ()

    def terminal_constraints(self, x):
        return np.zeros(0)

    def terminal_constraint_jacobian(self, x):
        return np.zeros((0, self.nx))

    def energy(self, x):
        n = self.n_links
        th, om = x[:n], x[n:]
        M = self._kappa * np.cos(th[:, None] - th[None, :]) + np.diag(self._inertia)
        return float(0.5 * om @ M @ om - (self._glever * np.cos(th)).sum())

    def disturbance(self, x):
        n = self.n_links
        E = np.zeros((2 * n, 2 * n))
        E[n:, n:] = self.e_rate * np.eye(n)
        return E

    def cost_weights(self):
        n = self.n_links
        Q = np.diag(np.concatenate([np.full(n, self.q_angle), np.full(n, self.q_rate)]))
        return Q, self.r_torque * np.eye(n), self.qn_scale * Q

    def upright(self):
        return np.concatenate([np.full(self.n_links, np.pi), np.zeros(self.n_links)])

    def reference(self, N):
        return np.tile(self.upright(), (N + 1, 1)), np.zeros((N, self.n_links))

    def device_spec(self):
        n = self.n_links
        return (DEV_PENDULUM, np.concatenate([[n, self.dt], self._kappa.ravel(), self._inertia, self._glever]),
                self._constraint_params())


@dataclass(frozen=True)
class Quadrotor12(_BoxObstacleModel):
    """12D quadrotor: p, euler (roll, pitch, yaw), v (world), omega (body); RK4.

    Thrusts u1..u4 on a plus frame: tau = (L(u2-u4), L(u3-u1), kappa(u1-u2+u3-u4)).
    """

    mass: float = 1.0
    arm: float = 0.2
    inertia: tuple = (0.01, 0.01, 0.02)
    kappa: float = 0.02
    dt: float = 0.02
    thrust_max: float = 6.0
    obstacles: tuple = ((1.0, 0.25, 0.3), (1.8, -0.4, 0.3), (2.6, 0.3, 0.3), (3.4, -0.2, 0.3),
                        (4.2, 0.35, 0.3))
    goal: tuple = (5.0, 0.0, 1.0, 0, 0, 0, 0, 0, 0, 0, 0, 0)
    q_diag: tuple = (2.0, 2.0, 2.0, 0.5, 0.5, 0.2, 0.2, 0.2, 0.2, 0.05, 0.05, 0.05)
    r_scale: float = 0.1
    qn_scale: float = 10.0
    e_scale: float = 5e-2
    nx: int = field(default=12, init=False)
    nu: int = field(default=4, init=False)

    def f_cont(self, x, u):
        vx, vy, vz = x[6], x[7], x[8]
        phi, th, psi = x[3], x[4], x[5]
        p, q, r = x[9], x[10], x[11]
        sf, cf, st, ct, sp, cp = np.sin(phi), np.cos(phi), np.sin(th), np.cos(th), np.sin(psi), np.cos(psi)
        T = u[0] + u[1] + u[2] + u[3]
        Jx, Jy, Jz = self.inertia
        tx = self.arm * (u[1] - u[3])
        ty = self.arm * (u[2] - u[0])
        tz = self.kappa * (u[0] - u[1] + u[2] - u[3])
        tt = st / ct
        return np.array([
            vx, vy, vz,
            p + sf * tt * q + cf * tt * r,
            cf * q - sf * r,
            (sf * q + cf * r) / ct,
            T / self.mass * (cf * st * cp + sf * sp),
            T / self.mass * (cf * st * sp - sf * cp),
            T / self.mass * (cf * ct) - GRAVITY,
            (tx - (Jz - Jy) * q * r) / Jx,
            (ty - (Jx - Jz) * p * r) / Jy,
            (tz - (Jy - Jx) * p * q) / Jz,
        ])

    def step(self, x, u):
        return rk4(self.f_cont, np.asarray(x), np.asarray(u), self.dt)

    def jacobians(self, x, u):
        return complex_step_jacobians(self.step, x, u)

    def hover_thrust(self):
        return self.mass * GRAVITY / 4.0

    def _u_bounds(self):
        return np.zeros(4), np.full(4, self.thrust_max)

    def disturbance(self, x):
        d = np.zeros(12)
        d[6:9] = self.e_scale
        return np.diag(d)

    def cost_weights(self):
        Q = np.diag(self.q_diag)
        return Q, self.r_scale * np.eye(4), self.qn_scale * Q

    def reference(self, N):
        return (np.tile(np.asarray(self.goal, float), (N + 1, 1)),
                np.full((N, 4), self.hover_thrust()))

    def device_spec(self):
        return (DEV_QUAD12, np.array([self.mass, self.arm, *self.inertia, self.kappa, self.dt], float),
                self._constraint_params())


class SyntheticLegged(_BoxObstacleModel):
    """Seeded stable nonlinear plant shaped like a legged robot.

    x+ = x + dt (A0 x + B0 u + c tanh(W x)); A = I + dt (A0 + c diag(1 - tanh^2(Wx)) W),
    B = dt B0.  A0 couples position-like and velocity-like halves
    (d/dt q = v, d/dt v = -K q - Dv v + ...), B0 drives the velocity half,
    W is a weak random coupling.  Constraints: |u| <= u_max plus obstacle rows
    on (x0, x1); terminal obstacle rows; E = e_scale on (x0, x1).
    """

    def __init__(self, nx: int = 61, nu: int = 12, seed: int = 0, dt: float = 0.02,
                 u_max: float = 5.0, obstacles=((0.6, 0.45, 0.25), (1.2, -0.45, 0.25)),
                 coupling: float = 0.5, e_scale: float = 0.004, goal_x0: float = 1.5):
        self.nx, self.nu, self.seed, self.dt = int(nx), int(nu), int(seed), float(dt)
        self.u_max = float(u_max)
        self.obstacles = tuple(tuple(float(v) for v in o) for o in obstacles)
        self.coupling = float(coupling)
        self.e_scale = float(e_scale)
        self.goal_x0 = float(goal_x0)
        rng = np.random.default_rng(self.seed)
        n, m = self.nx, self.nu
        h = n // 2
        A0 = np.zeros((n, n))
        A0[:h, h:2 * h] = np.eye(h)
        K = rng.uniform(0.5, 2.0, h)
        A0[h:2 * h, :h] = -np.diag(K) + 0.1 * rng.standard_normal((h, h)) / np.sqrt(h)
        A0[h:2 * h, h:2 * h] = -np.diag(rng.uniform(1.0, 3.0, h))
        if n > 2 * h:
            A0[n - 1, n - 1] = -0.5
        # positions 0, 1 are "base" coordinates: no stiffness, pure damping
        A0[h, 0] = 0.0
        A0[h + 1, 1] = 0.0
        B0 = np.zeros((n, m))
        B0[h:2 * h] = rng.standard_normal((h, m)) / np.sqrt(m)
        B0[h, :] += 1.0 / np.sqrt(m)
        B0[h + 1, :] -= 0.5 / np.sqrt(m)
        W = 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
        self.A0, self.B0, self.W = A0, B0, W
        q = np.full(n, 0.1)
        q[:2] = 5.0
        q[h:h + 2] = 0.5
        self._Q = np.diag(q)
        self._R = 0.05 * np.eye(m)
        self._QN = 10.0 * self._Q
        self._goal = np.zeros(n)
        self._goal[0] = self.goal_x0

    def step(self, x, u):
        x = np.asarray(x)
        u = np.asarray(u)
        return x + self.dt * (self.A0 @ x + self.B0 @ u + self.coupling * np.tanh(self.W @ x))

    def jacobians(self, x, u):
        s = 1.0 - np.tanh(self.W @ np.asarray(x, float)) ** 2
        A = np.eye(self.nx) + self.dt * (self.A0 + self.coupling * s[:, None] * self.W)
        return A, self.dt * self.B0

    def _u_bounds(self):
        return np.full(self.nu, -self.u_max), np.full(self.nu, self.u_max)

    def disturbance(self, x):
        d = np.zeros(self.nx)
        d[:2] = self.e_scale
        return np.diag(d)

    def cost_weights(self):
        return self._Q, self._R, self._QN

    def reference(self, N):
        return np.tile(self._goal, (N + 1, 1)), np.zeros((N, self.nu))

    def device_spec(self):
        return (DEV_SYNTH, np.concatenate([[self.dt, self.coupling], self.A0.ravel(), self.B0.ravel(),
                                           self.W.ravel()]), self._constraint_params())


def quadruped61(seed: int = 0, **kw) -> SyntheticLegged:
    """BASELINE cfg-D plant: 61D state, 12 torques."""
    return SyntheticLegged(61, 12, seed=seed, **kw)


def humanoid75(seed: int = 0, **kw) -> SyntheticLegged:
    """BASELINE cfg-E plant: 75D state, 19 torques."""
    kw.setdefault("u_max", 1.2)
    return SyntheticLegged(75, 19, seed=seed, **kw)


_MODELS = {"dubins": DubinsCar, "quadrotor": PlanarQuadrotor, "pendulum": NLinkPendulum,
           "quadrotor12": Quadrotor12, "synthetic": SyntheticLegged}


def make_model(model_id: str, **params) -> Model:
    """models.py:454-464."""
    try:
        cls = _MODELS[model_id]
    except KeyError:
        raise ValueError(f"unknown model id {model_id!r}") from None
    if "obstacles" in params:
        params["obstacles"] = tuple(tuple(o) for o in params["obstacles"])
    for key in ("goal", "masses", "lengths", "q_diag", "r_diag", "qn_diag"):
        if key in params and params[key] is not None:
            params[key] = tuple(params[key])
    return cls(**params)
