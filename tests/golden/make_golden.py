"""Generate the golden fixtures in tests/golden from the REFERENCE package.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is imported read-only; only its outputs (numbers) are stored.
Nothing in the test suite reads /root/reference at run time.
"""

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from chebchan import matrices as RM  # noqa: E402
from chebchan import solvers as RS  # noqa: E402
from chebchan import transforms as RT  # noqa: E402
from chebchan.mesh import PointFamily, Space, build_mesh, wavenumber_grid  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FAMS = list(PointFamily)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def z2_grid(n_y, n_z, l_y=2 * np.pi, l_z=np.pi):
    m = 2 * np.pi * np.fft.fftfreq(n_y, 1.0 / n_y) / l_y
    n = 2 * np.pi * np.fft.rfftfreq(n_z, 1.0 / n_z) / l_z
    return m[:, None] ** 2 + n[None, :] ** 2


def matrices_fixture():
    out = {}
    for n_x in (8, 16, 63, 64, 256):
        for fi, fam in enumerate(FAMS):
            m = RM.assemble(n_x, fam)
            key = f"nx{n_x}_f{fi}"
            out[key + "_mass_cheb"] = m.mass_cheb
            for name in ("mass_dir", "mass_bih", "mixed_mass", "stiff_bih", "deriv_dir_to_bih", "deriv_bih_to_dir"):
                mat = getattr(m, name)
                for off, dg in zip(mat.offsets, mat.diagonals):
                    out[f"{key}_{name}_{off}"] = dg
            for name in ("stiff_dir", "deriv_dir_to_cheb"):
                mat = getattr(m, name)
                for off, dg in zip(mat.banded.offsets, mat.banded.diagonals):
                    out[f"{key}_{name}_{off}"] = dg
                out[f"{key}_{name}_tail"] = mat.tail
            out[key + "_fourth_bih_diag"] = m.fourth_bih.diag
    np.savez_compressed(os.path.join(OUT, "matrices.npz"), **out)


def solver_fixture():
    """Small cases: full factors + solutions (real and complex RHS)."""
    out = {}
    meta = []
    cases = []
    for n_x in (16, 32, 63):
        for fi in (0, 1):
            cases.append((n_x, fi, 1 / 5200, 1e-5, np.array([0.0, 10.0, 200.0]) ** 2))
    cases.append((256, 0, 1 / 5200, 1e-5, np.array([5400.0]) ** 2))
    cases.append((64, 0, 0.01, 0.1, np.linspace(0.0, 400.0, 12).reshape(3, 4)))
    for ci, (n_x, fi, nu, dt, z2) in enumerate(cases):
        mats = RM.assemble(n_x, FAMS[fi])
        rng = np.random.default_rng(1000 + ci)
        key = f"c{ci}"
        out[key + "_z2"] = z2
        for op, build, nm in (("h", RS.build_helmholtz, mats.n_dir), ("b", RS.build_biharmonic, mats.n_bih)):
            lu = build(mats, nu, dt, z2)
            fr = rng.standard_normal((nm,) + z2.shape)
            fc = rng.standard_normal((nm,) + z2.shape) + 1j * rng.standard_normal((nm,) + z2.shape)
            out[f"{key}_{op}_rhs_real"] = fr
            out[f"{key}_{op}_rhs_cplx"] = fc
            out[f"{key}_{op}_x_real"] = lu.solve(fr)
            out[f"{key}_{op}_x_cplx"] = lu.solve(fc)
            names = ("low", "d", "e", "tail") if op == "h" else ("low2", "low4", "d", "e", "f", "a", "b")
            for nmf in names:
                for p in (0, 1):
                    out[f"{key}_{op}_{nmf}{p}"] = getattr(lu, nmf)[p]
        meta.append({"case": ci, "n_x": n_x, "family": fi, "nu": nu, "dt": dt, "z2_shape": list(z2.shape)})
    np.savez_compressed(os.path.join(OUT, "solvers.npz"), **out)
    return meta


def baseline_fixture():
    """BASELINE configs 1 and 2 (n_x = 63, 64 x 33 wavenumbers, nu = dt = 1e-3,
    RHS N(0,1) complex from default_rng(0), real part first): sha256 of the
    reference's full solution plus every 16th system verbatim."""
    mats = RM.assemble(63, PointFamily.GAUSS)
    z2 = z2_grid(64, 64)
    res = {}
    arrays = {}
    for op, build, nm in (("h", RS.build_helmholtz, mats.n_dir), ("b", RS.build_biharmonic, mats.n_bih)):
        rng = np.random.default_rng(0)
        f = rng.standard_normal((nm,) + z2.shape) + 1j * rng.standard_normal((nm,) + z2.shape)
        lu = build(mats, 1e-3, 1e-3, z2)
        x = lu.solve(f)
        res[op] = {"rhs_sha256": sha(f), "x_sha256": sha(x), "shape": list(x.shape)}
        flat = x.reshape(nm, -1)
        arrays[f"{op}_x_every16"] = flat[:, ::16]
        if op == "h":
            res[op]["factor_sha256"] = {f"{k}{p}": sha(getattr(lu, k)[p]) for k in ("low", "d", "e", "tail")
                                        for p in (0, 1)}
    np.savez_compressed(os.path.join(OUT, "baseline_c1c2.npz"), **arrays)
    return res


def transforms_fixture():
    out = {}
    for n_x in (8, 16, 32):
        for fi, fam in enumerate(FAMS):
            mesh = build_mesh(n_x, 8, 4, 2 * np.pi, np.pi, fam)
            rng = np.random.default_rng(7 * n_x + fi)
            u = rng.standard_normal(mesh.shape)
            key = f"nx{n_x}_f{fi}"
            out[key + "_u"] = u
            for space in Space:
                sc = list(Space).index(space)
                c = RT.forward_transform(RT.PhysicalField(u, mesh), space)
                out[f"{key}_s{sc}_fwd"] = c.data
                out[f"{key}_s{sc}_fsp"] = RT.forward_scalar_product(RT.PhysicalField(u, mesh), space).data
                out[f"{key}_s{sc}_inv"] = RT.inverse_transform(c).data
    # 1-D building blocks on a (n_x+1, 3) complex block
    for fi, fam in enumerate(FAMS):
        rng = np.random.default_rng(99 + fi)
        v = rng.standard_normal((13, 3)) + 1j * rng.standard_normal((13, 3))
        out[f"blk_f{fi}_v"] = v
        out[f"blk_f{fi}_cheb_scalar"] = RT.chebyshev_scalar(v, fam)
        out[f"blk_f{fi}_cheb_eval"] = RT.chebyshev_evaluate(v, fam)
        for space in (Space.DIRICHLET, Space.BIHARMONIC):
            sc = list(Space).index(space)
            out[f"blk_f{fi}_s{sc}_shen_scalar"] = RT.shen_scalar(v, fam, space)
            w = v[:13 - space.mode_drop]
            out[f"blk_f{fi}_s{sc}_expand"] = RT.shen_expand(w, space, 12)
            out[f"blk_f{fi}_s{sc}_mass"] = RT.mass_solve(w, space, 12, fam)
    np.savez_compressed(os.path.join(OUT, "transforms.npz"), **out)


def apply_fixture():
    """Reference structured apply (matrices.py apply) on seeded inputs."""
    out = {}
    names = ("mass_dir", "mass_bih", "mixed_mass", "stiff_dir", "stiff_bih", "fourth_bih", "deriv_dir_to_bih",
             "deriv_bih_to_dir", "deriv_dir_to_cheb")
    for n_x in (16, 33):
        for fi, fam in enumerate(FAMS):
            m = RM.assemble(n_x, fam)
            for name in names:
                M = getattr(m, name)
                rng = np.random.default_rng([n_x, fi, names.index(name)])
                x = rng.standard_normal((M.shape[1], 6)) + 1j * rng.standard_normal((M.shape[1], 6))
                out[f"nx{n_x}_f{fi}_{name}_x"] = x
                out[f"nx{n_x}_f{fi}_{name}_y"] = M.apply(x)
    np.savez_compressed(os.path.join(OUT, "apply.npz"), **out)


def rhs_fixture():
    """Reference ChannelStepper._ab2 / assemble_rhs_u / assemble_rhs_g on a
    seeded state (n_x = 16, 8 x 8 plane, both families)."""
    from chebchan.stepper import ChannelStepper, FlowState, StepperConfig
    from chebchan.transforms import SpectralField

    out = {}
    for fi, fam in enumerate(FAMS):
        mesh = build_mesh(16, 8, 8, 2 * np.pi, np.pi, fam)
        st = ChannelStepper(mesh, StepperConfig(nu=1e-2, dt=1e-3))
        gd, gb = wavenumber_grid(mesh, Space.DIRICHLET), wavenumber_grid(mesh, Space.BIHARMONIC)
        rng = np.random.default_rng(50 + fi)

        def cf(grid):
            shp = (grid.n_modes,) + mesh.spectral_shape_yz
            return SpectralField(rng.standard_normal(shp) + 1j * rng.standard_normal(shp), grid, mesh)

        u, v, w, g = cf(gb), cf(gd), cf(gd), cf(gd)
        hc = tuple(cf(gd) for _ in range(3))
        hp = tuple(cf(gd) for _ in range(3))
        state = FlowState(u, v, w, g, hc, hp, 0.0, 0.0, 0)
        h_ab = st._ab2(state)
        key = f"f{fi}"
        out[key + "_u"], out[key + "_g"] = u.data, g.data
        for i in range(3):
            out[f"{key}_hc{i}"], out[f"{key}_hp{i}"], out[f"{key}_hab{i}"] = hc[i].data, hp[i].data, h_ab[i]
        out[key + "_rhs_u"] = st.assemble_rhs_u(state, h_ab)
        out[key + "_rhs_g"] = st.assemble_rhs_g(state, h_ab)
        out[key + "_m"], out[key + "_n"], out[key + "_z2"] = st.m, st.n, st.z2
        # nonlinear term of the same state (dealiased)
        nl = st.compute_nonlinear(state)
        for i in range(3):
            out[f"{key}_nl{i}"] = nl[i].data
        out[key + "_v"], out[key + "_w"], out[key + "_mask"] = v.data, w.data, st.mask
        # velocity recovery lines of stepper.py:296-303 with the reference's own functions
        f_scal = st.mats.deriv_bih_to_dir.apply(u.data)
        f_hat = RT.mass_solve(f_scal, Space.DIRICHLET, mesh.n_x, mesh.family)
        safe_z2 = np.where(st.z2 > 0, st.z2, 1.0)
        out[key + "_vrec"] = (1j * st.m * f_hat + 1j * st.n * g.data) / safe_z2
        out[key + "_wrec"] = (1j * st.n * f_hat - 1j * st.m * g.data) / safe_z2
        # one full reference time step from this state, both forcings
        from chebchan.stepper import Forcing

        for tag, cfg in (("fb", StepperConfig(nu=1e-2, dt=1e-3, beta=0.5)),
                         ("cf", StepperConfig(nu=1e-2, dt=1e-3, forcing=Forcing.CONSTANT_FLUX, target_flux=0.3))):
            stp = ChannelStepper(mesh, cfg)
            new = stp.step(FlowState(u, v, w, g, hc, hp, 0.25, 1.5, 7))
            for nm in ("u_hat", "v_hat", "w_hat", "g_hat"):
                out[f"{key}_{tag}_{nm}"] = getattr(new, nm).data
            for i in range(3):
                out[f"{key}_{tag}_hcur{i}"] = new.h_curr[i].data
            out[f"{key}_{tag}_beta"] = np.array(new.beta)
        # a reference checkpoint of the same state (wire-format fixture)
        from chebchan.stepper import save_checkpoint

        save_checkpoint(os.path.join(OUT, f"checkpoint_f{fi}.bin"),
                        FlowState(u, v, w, g, hc, hp, 0.25, 1.5, 7), StepperConfig(nu=1e-2, dt=1e-3))
    np.savez_compressed(os.path.join(OUT, "rhs.npz"), **out)


def big_fixture():
    """Headline-size pins: sha256 of every assemble() table at n_x = 1024 and
    2048 (config 4 / config 5's largest N), and the reference's 3-D forward
    and inverse transforms at n_x = 512 and 1024 (Gauss and Lobatto) on a thin
    (n_y, n_z) = (4, 2) plane, where the biharmonic forward map is most
    ill-conditioned."""
    tables = {}
    for n_x in (1024, 2048):
        for fi, fam in enumerate(FAMS):
            m = RM.assemble(n_x, fam)
            key = f"nx{n_x}_f{fi}"
            tables[key + "_mass_cheb"] = sha(m.mass_cheb)
            for name in ("mass_dir", "mass_bih", "mixed_mass", "stiff_bih", "deriv_dir_to_bih", "deriv_bih_to_dir"):
                mat = getattr(m, name)
                for off, dg in zip(mat.offsets, mat.diagonals):
                    tables[f"{key}_{name}_{off}"] = sha(dg)
            for name in ("stiff_dir", "deriv_dir_to_cheb"):
                mat = getattr(m, name)
                for off, dg in zip(mat.banded.offsets, mat.banded.diagonals):
                    tables[f"{key}_{name}_{off}"] = sha(dg)
                tables[f"{key}_{name}_tail"] = sha(mat.tail)
            tables[key + "_fourth_bih_diag"] = sha(m.fourth_bih.diag)
    out = {}
    for n_x in (512, 1024):
        for fi, fam in enumerate(FAMS):
            mesh = build_mesh(n_x, 4, 2, 2 * np.pi, np.pi, fam)
            u = np.random.default_rng(n_x + fi).uniform(-1, 1, mesh.shape)
            key = f"nx{n_x}_f{fi}"
            out[key + "_u"] = u
            for space in (Space.DIRICHLET, Space.BIHARMONIC):
                sc = list(Space).index(space)
                c = RT.forward_transform(RT.PhysicalField(u, mesh), space)
                out[f"{key}_s{sc}_fwd"] = c.data
                out[f"{key}_s{sc}_inv"] = RT.inverse_transform(c).data
    np.savez_compressed(os.path.join(OUT, "big_transforms.npz"), **out)
    with open(os.path.join(OUT, "big_tables.json"), "w") as fh:
        json.dump(tables, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    if "--big-only" in sys.argv:
        big_fixture()
        sys.exit(0)
    if "--apply-only" in sys.argv:
        apply_fixture()
        sys.exit(0)
    if "--rhs-only" in sys.argv:
        rhs_fixture()
        sys.exit(0)
    matrices_fixture()
    meta = solver_fixture()
    base = baseline_fixture()
    transforms_fixture()
    apply_fixture()
    rhs_fixture()
    big_fixture()
    with open(os.path.join(OUT, "golden_meta.json"), "w") as fh:
        json.dump({"solver_cases": meta, "baseline": base,
                   "generator": "tests/golden/make_golden.py from /root/reference/pkg/src (chebchan 0.1.0)",
                   "numpy": np.__version__}, fh, indent=1)
    print("golden fixtures written to", OUT)
