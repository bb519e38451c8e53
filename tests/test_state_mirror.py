"""CPU: the device-backed SimState view downloads fields lazily and writes back only
what the caller modified (no GPU: a fake scene stands in for the C ABI)."""

import numpy as np

from paper_2403_19272_b200.stepper import DeviceSimState


class _FakeSim:
    def __init__(self, n=5):
        self._step_index = 3
        self.dev = {k: np.random.default_rng(i).standard_normal((n, 3)) for i, k in enumerate(DeviceSimState.FIELDS)}
        self.downloads = []

    def _download(self, name):
        self.downloads.append(name)
        return self.dev[name].copy()


def test_lazy_fields_and_dirty_tracking():
    sim = _FakeSim()
    st = DeviceSimState(sim)
    assert st.step_index == 3 and sim.downloads == []
    x = st.x
    assert sim.downloads == ["x"] and np.array_equal(x, sim.dev["x"])
    assert st.x is x and sim.downloads == ["x"]            # cached
    assert not any(st.dirty(k) for k in DeviceSimState.FIELDS)
    st.x_dot[:] = (0.0, 0.0, -1.0)                         # reference tests/test_stepper.py:58
    assert st.dirty("x_dot") and not st.dirty("x")
    view = st.x[1:3]
    view[:] = 7.0                                          # writes through a view
    assert st.dirty("x") and np.all(st.x[1:3] == 7.0)
    st.delta_f = np.ones((5, 3))                           # assignment marks dirty
    assert st.dirty("delta_f") and not st.dirty("x_prev")
    assert "x_prev" not in sim.downloads


def test_arithmetic_results_are_plain_arrays():
    sim = _FakeSim()
    st = DeviceSimState(sim)
    y = st.x + 1.0
    y[:] = 0.0                                            # a derived array is not state
    assert not st.dirty("x")


def test_inplace_ufunc_marks_dirty():
    sim = _FakeSim()
    st = DeviceSimState(sim)
    v = st.x_dot
    v *= 2.0
    assert st.dirty("x_dot")
    np.add(st.x_prev, 1.0, out=st.x_prev)
    assert st.dirty("x_prev")


def test_every_write_path_is_tracked_or_loud():
    """np.copyto / .fill / np.add.at / np.put reach the device; a write
    through an untracked plain view raises instead of being silently lost."""
    import pytest

    sim = _FakeSim()
    st = DeviceSimState(sim)
    np.copyto(st.x, np.zeros((5, 3)))
    assert st.dirty("x") and not st.x.any()
    st.x_dot.fill(2.0)
    assert st.dirty("x_dot") and (st.x_dot == 2.0).all()
    np.add.at(st.delta_f, [0, 0], 1.0)
    assert st.dirty("delta_f")
    np.put(st.x_prev, [0], 9.0)
    assert st.dirty("x_prev") and st.x_prev[0, 0] == 9.0
    fresh = DeviceSimState(sim)
    with pytest.raises(ValueError, match="read-only"):
        np.asarray(fresh.x)[0] = 1.0
    assert not fresh.dirty("x")
    row = fresh.x[2]                                      # a view taken before the write
    row[1] = 4.0
    assert fresh.dirty("x") and fresh.x[2, 1] == 4.0
    y = fresh.x_dot.copy()                                # copies are writeable
    y[0] = 1.0
