"""CPU: the C-ABI library builds, loads and exports every symbol the header
declares (no compute calls - there is no GPU here)."""

import os
import re

import pytest

from paper_2403_19272_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "clothsim_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cs_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(_lib.EXPORTED)


def test_library_exports_every_symbol():
    from paper_2403_19272_b200 import build

    path = build.build()
    lib = _lib.load(path)
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.cs_version().startswith(b"clothsim_b200")


def test_struct_layouts_match_header():
    """ctypes mirrors of the header structs: field names in declaration order."""
    text = open(HEADER).read()
    body = text[text.index("typedef struct {\n    int n_cloth"):text.index("} cs_scene_desc;")]
    names = re.findall(r"\*?\s*\*?([A-Za-z_0-9]+)\s*[,;]", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert [f[0] for f in _lib.SceneDesc._fields_] == names


def test_no_cpu_fallback_without_library(tmp_path):
    with pytest.raises(RuntimeError):
        _lib._lib = None
        _lib.load(str(tmp_path / "missing.so"))
    _lib._lib = None


def _struct_fields(text, tail):
    end = text.index("} " + tail + ";")
    start = text.rindex("typedef struct {", 0, end)
    body = re.sub(r"/\*.*?\*/", "", text[start + len("typedef struct {"):end], flags=re.S)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        # "double t_a, t_b" / "double outer_deltas[64]" / "long long a, b"
        parts = decl.split(",")
        first = parts[0].split()
        names.append(re.sub(r"\[.*\]", "", first[-1]).lstrip("*"))
        names.extend(re.sub(r"\[.*\]", "", p.strip()).lstrip("*") for p in parts[1:])
    return names


def test_report_and_config_layouts_match_header():
    """cs_step_report / cs_step_config ctypes mirrors: the header's fields in order
    (a mismatch would silently shift every report field after it)."""
    text = open(HEADER).read()
    assert [f[0] for f in _lib.StepReportC._fields_] == _struct_fields(text, "cs_step_report")
    assert [f[0] for f in _lib.StepConfigC._fields_] == _struct_fields(text, "cs_step_config")
