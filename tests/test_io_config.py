"""Frame/metrics I/O: config files, OBJ text and metrics rows against
the reference's own outputs (tests/golden/io.npz, made by running the reference CLI)."""
import numpy as np
import pytest

from conftest import golden
from paper_2403_19272_b200.cli import METRIC_FIELDS, ObjFormatter, metrics_row
from paper_2403_19272_b200.sceneconfig import ConfigError, SceneConfig, parse_config, serialize_config
from paper_2403_19272_b200.stepconfig import StepReport


def test_config_roundtrip_matches_reference():
    g = golden("io.npz")
    cfg = parse_config(str(g["config_in"]))
    assert serialize_config(cfg) == str(g["config_roundtrip"])
    assert cfg.solver.gravity == (0.0, -9.8, 0.0) and cfg.solver.samples == 6
    assert parse_config(serialize_config(cfg)) == cfg


def test_config_defaults_and_errors():
    assert parse_config("") == SceneConfig()
    with pytest.raises(ConfigError):
        parse_config("[scene]\nkinds = 'x'\n")
    with pytest.raises(ConfigError):
        parse_config("[nope]\na = 1\n")
    with pytest.raises(ConfigError):
        parse_config("scene = 3\n")
    with pytest.raises(ConfigError):
        parse_config("[solver]\nalpha = 2.0\n")        # StepConfig validation
    with pytest.raises(ConfigError):
        parse_config("[scene\n")


def test_obj_text_matches_reference_save_obj(tmp_path):
    g = golden("io.npz")
    path = tmp_path / "a.obj"
    ObjFormatter(g["fixed_tris"]).write(path, g["fixed_verts"])
    assert path.read_text() == str(g["fixed_obj"])


def test_metrics_row_format():
    g = golden("io.npz")
    lines = str(g["metrics"]).splitlines()
    assert lines[0].split(",") == METRIC_FIELDS
    rep = StepReport(lg_iterations=1, outer_loops=1, toi_exit=1.0, active_pairs=0,
                     timings={k: 0.5 for k in ("warm_start", "local", "global", "smoothing", "broad",
                                                "narrow_partial", "narrow_full")})
    row = [str(v) for v in metrics_row(1, rep)]
    assert row[:7] == lines[1].split(",")[:7]
    assert row[7:] == ["0.500"] * 7
