"""Frame/metrics I/O on the device path: `simulate` with async frame
snapshots (cs_frame_async) against the reference CLI's own run (tests/golden/io.npz)."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _parse_obj(text):
    v = np.array([[float(t) for t in ln.split()[1:]] for ln in text.splitlines() if ln.startswith("v ")])
    f = [ln for ln in text.splitlines() if ln.startswith("f ")]
    return v, f


def _run(tmp_path, text, **kw):
    from paper_2403_19272_b200.cli import simulate
    from paper_2403_19272_b200.sceneconfig import parse_config

    out = tmp_path / "out"
    cfg = parse_config(text.replace("[output]\n", f'[output]\ndirectory = "{out}"\n'))
    assert simulate(cfg, **kw) == 0
    return out


def test_simulate_matches_reference_cli(cuda, tmp_path):
    g = golden("io.npz")
    out = _run(tmp_path, str(g["config_in"]))
    frames = sorted(p.name for p in out.glob("frame_*.obj"))
    assert frames == list(g["frames"])
    for name, ref_text in zip(frames, g["objs"]):
        v, f = _parse_obj((out / name).read_text())
        rv, rf = _parse_obj(str(ref_text))
        assert f == rf
        assert np.abs(v - rv).max() <= 2e-9          # 9-decimal text of trajectories equal to 1e-9 m
    ours = (out / "metrics.csv").read_text().splitlines()
    ref = str(g["metrics"]).splitlines()
    assert ours[0] == ref[0] and len(ours) == len(ref)
    for a, b in zip(ours[1:], ref[1:]):
        assert a.split(",")[:7] == b.split(",")[:7]   # counters, toi, flags; timings differ
    strip = lambda t: [ln for ln in t.splitlines() if not ln.startswith("directory")]  # noqa: E731
    assert strip((out / "config.toml").read_text()) == strip(str(g["config_written"]))


def test_async_frames_equal_synchronous_state(cuda, tmp_path):
    """Every frame written through the snapshot ring (stride 1: both slots and both
    host buffers recycled every step) is the state the step produced."""
    import paper_2403_19272_b200 as P
    from paper_2403_19272_b200.cli import ObjFormatter, build_from_config
    from paper_2403_19272_b200.sceneconfig import parse_config

    text = ('name = "s"\nsteps = 6\n\n[scene]\nkind = "sphere_drape"\nresolution = 12\nsize = 0.3\n\n'
            '[solver]\nh = 0.005\n\n[output]\nframe_stride = 1\n')
    out = _run(tmp_path, text)
    sim = build_from_config(parse_config(text))
    fmt = ObjFormatter(sim.mesh.triangles)
    for step in range(7):
        if step:
            sim.step()
        ref = tmp_path / "ref.obj"
        fmt.write(ref, sim.state.x)
        assert (out / f"frame_{step:06d}.obj").read_text() == ref.read_text(), step
    assert isinstance(P.StepConfig(), P.StepConfig)
