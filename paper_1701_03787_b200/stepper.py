"""One time step of the reference's channel stepper on the device, composed
of this package's kernels (the callers either side of the
solves; reference ``stepper.py:102-346``, ``ChannelStepper.step``).

``DeviceStepper(mesh, config).step(state)`` = ``ChannelStepper.step``:

1. nonlinear term H = u x omega (``nonlinear.NonlinearTerm``, 8 inverse +
   3 forward transforms, stepper.py:148-185);
2. AB2 + right-hand sides of the implicit updates (``rhs.RhsAssembler``,
   :189-219);
3. the batched biharmonic and Helmholtz solves (``solvers``, :293-294);
4. divergence variable and v, w recovery (``recover.VelocityRecovery``,
   :296-303);
5. the mean-flow (m = n = 0) momentum equations with the driving gradient
   and optional constant-flux control (:305-330) -- one-system Helmholtz
   solves on the device.

All state stays on the device (torch CUDA tensors inside the
``SpectralField`` containers).  The stepper itself is not part of the
hot-path scope; this class is the composition that validates the pieces
together against the reference (tests/test_stepper_gpu.py) and times a
whole step (bench.py --config step).
"""

from __future__ import annotations

import numpy as np

from . import operators, solvers
from .checkpoint import FlowState
from .matrices import assemble
from .mesh import Space, wavenumber_grid
from .nonlinear import NonlinearTerm
from .recover import VelocityRecovery
from .rhs import RhsAssembler
from .transforms import SpectralField

__all__ = ["DeviceStepper", "dirichlet_integral_weights"]


def dirichlet_integral_weights(n_modes: int) -> np.ndarray:
    """Exact integrals of the Dirichlet basis functions (stepper.py:83-91)."""
    ell = np.arange(n_modes)
    out = np.zeros(n_modes)
    even = ell % 2 == 0
    le = ell[even].astype(float)
    out[even] = 2 / (1 - le ** 2) - 2 / (1 - (le + 2) ** 2)
    return out


def _forcing(config) -> str:
    f = getattr(config, "forcing", "fixed-beta")
    return getattr(f, "value", f)


class DeviceStepper:
    """Device counterpart of ``ChannelStepper`` (constructor stepper.py:103-126)."""

    def __init__(self, mesh, config):
        import torch

        from ._device import device

        self.dev = device()
        self.mesh, self.config = mesh, config
        self.mats = assemble(mesh.n_x, mesh.family)
        self.grid_dir = wavenumber_grid(mesh, Space.DIRICHLET)
        self.grid_bih = wavenumber_grid(mesh, Space.BIHARMONIC)
        self.m = self.grid_dir.m_scaled[:, None]
        self.n = self.grid_dir.n_scaled[None, :]
        self.z2 = self.grid_dir.z2()
        nu, dt = config.nu, config.dt
        self.helmholtz = solvers.build_helmholtz(self.mats, nu, dt, self.z2)
        self.biharmonic = solvers.build_biharmonic(self.mats, nu, dt, self.z2)
        self.helmholtz_mean = solvers.build_helmholtz(self.mats, nu, dt, np.zeros(1))
        self.mask = self._spectral_mask()
        self.flux_weights = dirichlet_integral_weights(self.mats.n_dir)
        e0 = np.zeros((self.mats.n_dir, 1))
        e0[0, 0] = np.pi * mesh.n_y * mesh.n_z
        self.beta_response = -dt * self.helmholtz_mean.solve(e0)[:, 0]
        self.flux_sensitivity = float(self.flux_weights @ self.beta_response) / (mesh.n_y * mesh.n_z)
        self._fw = torch.from_numpy(self.flux_weights).to(self.dev)
        self._br = torch.from_numpy(self.beta_response).to(self.dev)
        self.nonlinear = NonlinearTerm(self.mats, mesh, self.m, self.n, self.mask)
        self.rhs = RhsAssembler(self.mats, nu, dt, self.z2, self.m, self.n)
        self.recovery = VelocityRecovery(self.mats, self.z2, self.m, self.n)

    def _spectral_mask(self) -> np.ndarray:
        """Dealiasing / Nyquist mask (stepper.py:130-140)."""
        n_y, n_z = self.mesh.n_y, self.mesh.n_z
        m_idx = np.fft.fftfreq(n_y, 1.0 / n_y).astype(int)[:, None]
        n_idx = np.arange(n_z // 2 + 1)[None, :]
        keep = (np.abs(m_idx) != n_y // 2) & (n_idx != n_z // 2)
        if getattr(self.config, "dealias", True):
            keep = keep & (np.abs(m_idx) < max(n_y // 3, 1)) & (n_idx < max(n_z // 3, 1))
        return keep

    def to_device(self, state):
        """A state with numpy fields -> the same state on the device."""
        import torch

        def f(x):
            d = x.data if hasattr(x.data, "is_cuda") else torch.from_numpy(np.ascontiguousarray(x.data))
            return SpectralField(d.to(self.dev, torch.complex128), x.grid, x.mesh)

        return FlowState(f(state.u_hat), f(state.v_hat), f(state.w_hat), f(state.g_hat),
                         tuple(f(h) for h in state.h_curr), tuple(f(h) for h in state.h_prev),
                         state.beta, state.t, state.kappa)

    def compute_nonlinear(self, state) -> tuple:
        """Dirichlet coefficients of H = u x omega, masked (stepper.py:148-185)."""
        h = self.nonlinear(state.u_hat.data, state.v_hat.data, state.w_hat.data, state.g_hat.data)
        return tuple(SpectralField(x, self.grid_dir, self.mesh) for x in h)

    def capture(self, state):
        """CUDA-graph a step that advances ``state`` IN PLACE (fixed-beta
        forcing only: constant-flux control reads the flux back to the host).

        Returns ``replay()``; each call advances the static state by one step
        (u, v, w, g, h_curr, h_prev updated on the device; t and kappa are
        advanced on ``state`` itself).  One graph launch replaces the ~100
        kernel launches and host work of ``step`` -- worth it on small meshes,
        where a step is launch-bound; on the config-3 mesh a step is GPU-bound
        and the in-place state copies make the graph ~10% slower (7.8 vs
        7.1 ms), so the bench times the eager step."""
        import torch

        if _forcing(self.config) != "fixed-beta":
            raise ValueError("graph capture needs fixed-beta forcing (constant flux syncs with the host)")
        fields = [state.u_hat.data, state.v_hat.data, state.w_hat.data, state.g_hat.data,
                  *(h.data for h in state.h_curr), *(h.data for h in state.h_prev)]
        if not all(getattr(f, "is_cuda", False) for f in fields):
            raise ValueError("capture needs the state on the device (DeviceStepper.to_device)")

        def body():
            new = self.step(state)
            for h_old, h_cur in zip(state.h_prev, state.h_curr):
                h_old.data.copy_(h_cur.data)
            for h_cur, h_new in zip(state.h_curr, new.h_curr):
                h_cur.data.copy_(h_new.data)
            state.u_hat.data.copy_(new.u_hat.data)
            state.v_hat.data.copy_(new.v_hat.data)
            state.w_hat.data.copy_(new.w_hat.data)
            state.g_hat.data.copy_(new.g_hat.data)

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        saved = [f.clone() for f in fields]
        with torch.cuda.stream(side):  # warm-up outside the graph (plans, caches, scratch)
            body()
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            body()
        for f, g in zip(fields, saved):  # undo the warm-up and capture side effects
            f.copy_(g)
        del saved

        def replay():
            graph.replay()
            state.t += self.config.dt
            state.kappa += 1

        replay.graph = graph
        return replay

    def step(self, state):
        """Advance one time step (stepper.py:286-346); device state in and out."""
        import torch

        mesh, cfg, mats = self.mesh, self.config, self.mats
        nu, dt = cfg.nu, cfg.dt
        h_new = self.compute_nonlinear(state)
        h_curr = tuple(h.data for h in h_new)
        h_prev = tuple(h.data for h in state.h_curr)
        u_new = self.biharmonic.solve(self.rhs.rhs_u(state.u_hat.data, h_curr, h_prev))
        g_new = self.helmholtz.solve(self.rhs.rhs_g(state.g_hat.data, h_curr, h_prev))
        v_new, w_new = self.recovery(u_new, g_new)
        # mean (m = n = 0) momentum equations with the driving gradient
        beta = cfg.beta if _forcing(cfg) == "fixed-beta" else state.beta

        def mean_rhs(vec, h_comp):
            rhs = -(nu * dt / 2) * operators.apply(mats.stiff_dir, vec)
            rhs += operators.apply(mats.mass_dir, vec)
            rhs += dt * operators.apply(mats.mass_dir, h_comp)
            return rhs

        v0 = state.v_hat.data[:, 0:1, 0].contiguous()
        w0 = state.w_hat.data[:, 0:1, 0].contiguous()
        hy0 = (1.5 * h_curr[1][:, 0:1, 0] - 0.5 * h_prev[1][:, 0:1, 0]).contiguous()
        hz0 = (1.5 * h_curr[2][:, 0:1, 0] - 0.5 * h_prev[2][:, 0:1, 0]).contiguous()
        rhs_v0 = mean_rhs(v0, hy0)
        rhs_v0[0] -= dt * beta * np.pi * mesh.n_y * mesh.n_z
        rhs_w0 = mean_rhs(w0, hz0)
        v0_new = self.helmholtz_mean.solve(rhs_v0)
        w0_new = self.helmholtz_mean.solve(rhs_w0)
        if _forcing(cfg) == "constant-flux":
            scale = mesh.n_y * mesh.n_z
            flux = float(torch.dot(self._fw, v0_new[:, 0].real)) / scale
            delta = (cfg.target_flux - flux) / self.flux_sensitivity
            v0_new = v0_new + delta * self._br[:, None]
            beta = beta + delta
        v_new[:, 0, 0] = v0_new[:, 0]
        w_new[:, 0, 0] = w0_new[:, 0]
        return FlowState(
            u_hat=SpectralField(u_new, self.grid_bih, mesh),
            v_hat=SpectralField(v_new, self.grid_dir, mesh),
            w_hat=SpectralField(w_new, self.grid_dir, mesh),
            g_hat=SpectralField(g_new, self.grid_dir, mesh),
            h_curr=h_new,
            h_prev=state.h_curr,
            beta=beta,
            t=state.t + dt,
            kappa=state.kappa + 1,
        )
