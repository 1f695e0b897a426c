"""Diagnostics / snapshot writers (reference output.py:1-99; SURVEY.md §8(f)
rank 3).  CPU: the text formats are byte-identical to the reference writers
on the reference's own states (golden `output_sod`).  GPU: a device run
writes the same diagnostics up to fp64 round-off, and two identical device
runs write identical bytes (test_acceptance.py:354-366)."""

import types

import numpy as np
import pytest

from paper_1808_03788_b200 import output
from paper_1808_03788_b200.basis import basis_tables
from paper_1808_03788_b200.mesh import CartesianMesh
from paper_1808_03788_b200.systems import make_system


def _history(g):
    return [{"step": int(s), "time": float(t), "dt": float(d), "totals": tot,
             "limited_fraction": float(f)}
            for s, t, d, tot, f in zip(g["steps"], g["times"], g["dts"], g["totals"], g["fracs"])]


def _fake_sim(mesh, system, degree, u, t, step):
    return types.SimpleNamespace(mesh=mesh, system=system, tables=basis_tables(degree), u=u,
                                 t=float(t), step_count=int(step))


def test_diagnostics_csv_matches_reference_bytes(golden):
    g = golden("output_sod")
    names = tuple(str(n) for n in g["names"])
    assert names == make_system("euler", 1).quantity_names
    assert output.diagnostics_csv(_history(g), names) == str(g["diag_csv"])


def test_snapshots_match_reference_bytes(golden):
    g = golden("output_sod")
    sim = _fake_sim(CartesianMesh([(0, 1)], (50,)), make_system("euler", 1), 2, g["u"], g["t"],
                    g["step_count"])
    assert output.fields_csv(sim) == str(g["fields_csv"])
    assert output.fields_vtk(sim) == str(g["fields_vtk"])
    sim2 = _fake_sim(CartesianMesh([(0, 10), (0, 10)], (4, 3)), make_system("euler", 2), 2,
                     g["u2"], g["t2"], 1)
    assert output.fields_vtk(sim2) == str(g["vtk2"])
    assert output.fields_csv(sim2) == str(g["csv2"])


def test_write_files_and_tdu(tmp_path, golden):
    g = golden("output_sod")
    names = make_system("euler", 1).quantity_names
    path = output.write_diagnostics(str(tmp_path / "diagnostics.csv"), _history(g), names)
    assert open(path).read() == str(g["diag_csv"])
    sim = _fake_sim(CartesianMesh([(0, 1)], (50,)), make_system("euler", 1), 2, g["u"], g["t"],
                    g["step_count"])
    p = output.write_snapshot(sim, str(tmp_path), "run", "vtk")
    assert p.endswith(f"run_{int(g['step_count']):06d}.vtk")
    assert open(p).read() == str(g["fields_vtk"])
    assert output.throughput_per_dof(1.25, 4096, 20, 4, 3) == float(g["tdu"])
    with pytest.raises(ValueError):
        output.throughput_per_dof(1.0, 0, 3, 2, 1)


@pytest.mark.gpu
def test_device_run_diagnostics(golden, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1808_03788_b200 as pkg

    g = golden("output_sod")
    names = make_system("euler", 1).quantity_names
    blobs = []
    for _ in range(2):
        system = pkg.make_system("euler", 1)
        sim = pkg.Simulation(pkg.CartesianMesh([(0, 1)], (50,)), system, 2, 0.15,
                             boundary="outflow", use_limiter=True)
        sim.project_initial_condition(pkg.build_problem("sod", system)[0])
        sim.run(np.inf, max_steps=8)
        blobs.append(output.diagnostics_csv(sim.history, names))
    assert blobs[0] == blobs[1]
    np.testing.assert_allclose([h["dt"] for h in sim.history], g["dts"], rtol=1e-12)
    np.testing.assert_allclose([h["time"] for h in sim.history], g["times"], rtol=1e-12)
    np.testing.assert_allclose(np.array([h["totals"] for h in sim.history]), g["totals"],
                               rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose([h["limited_fraction"] for h in sim.history], g["fracs"])
    u = sim.u.cpu().numpy()
    assert np.max(np.abs(u - g["u"])) / np.max(np.abs(g["u"])) <= 1e-10
    p = output.write_snapshot(sim, str(tmp_path), "sod", "csv")
    assert open(p).read().count("\n") == 50 * 3 + 1
    avg = output.cell_averages(sim)
    assert avg.shape == (50, 3)
