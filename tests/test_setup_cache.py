"""On-disk HostMesh cache (paper_2108_05110_b200/setup_cache.py): a loaded entry equals a fresh
build array for array; any input change gives a new key; broken entries rebuild."""
import dataclasses
import os

import numpy as np
import pytest

from paper_2108_05110_b200 import engine as E
from paper_2108_05110_b200 import setup_cache as SC
from paper_2108_05110_b200.problems import build_case


def _same(a, b):
    for k, v in vars(a).items():
        if k in ("disc", "plan", "_allkey"):
            continue
        w = getattr(b, k)
        if isinstance(v, np.ndarray):
            assert v.dtype == w.dtype and np.array_equal(v, w), k
        else:
            assert v == w, k
    for f in dataclasses.fields(a.plan):
        v, w = getattr(a.plan, f.name), getattr(b.plan, f.name)
        if f.name == "schedule":
            assert set(v) == set(w)
            for k in v:
                assert np.array_equal(np.asarray(v[k]), np.asarray(w[k])), k
        elif isinstance(v, np.ndarray):
            assert v.dtype == w.dtype and np.array_equal(v, w), f.name
        else:
            assert v == w, f.name


@pytest.fixture
def cache(tmp_path, monkeypatch):
    monkeypatch.setenv("ENS_SETUP_CACHE", str(tmp_path))
    monkeypatch.setenv("ENS_SETUP_CACHE_MIN_DOFS", "0")
    return tmp_path


@pytest.mark.parametrize("case,over", [("C2", dict(n=16)), ("C4", dict(k=2, length=10.0))])
def test_cached_equals_fresh(cache, case, over):
    disc, _, _ = build_case(case, steps=1, **over)
    cold = SC.host_mesh(disc)
    assert SC.last["hit"] is False and SC.last["cached"] is True
    assert (cache / SC.last["key"] / "meta.json").exists()
    disc2, _, _ = build_case(case, steps=1, **over)
    warm = SC.host_mesh(disc2)
    assert SC.last["hit"] is True
    _same(E.HostMesh(disc2), warm)
    _same(cold, warm)


def test_key_tracks_inputs(cache):
    d1, _, _ = build_case("C2", n=8, steps=1)
    d2, _, _ = build_case("C2", n=8, steps=1)
    d3, _, _ = build_case("C2", n=10, steps=1)
    d4, _, _ = build_case("C2", n=8, steps=1, pressure="disc")
    assert SC.mesh_key(d1) == SC.mesh_key(d2)
    assert len({SC.mesh_key(d) for d in (d1, d3, d4)}) == 3
    d2.pin_pressure = False                       # constrained rows change
    assert SC.mesh_key(d2) != SC.mesh_key(d1)


def test_broken_entry_rebuilds(cache):
    disc, _, _ = build_case("C2", n=8, steps=1)
    SC.host_mesh(disc)
    key = SC.last["key"]
    os.remove(cache / key / "hm.s_mass.npy")
    d2, _, _ = build_case("C2", n=8, steps=1)
    hm = SC.host_mesh(d2)
    assert SC.last["hit"] is False
    _same(E.HostMesh(d2), hm)


def test_disabled_and_small(monkeypatch, tmp_path):
    monkeypatch.setenv("ENS_SETUP_CACHE", "off")
    disc, _, _ = build_case("C2", n=8, steps=1)
    SC.host_mesh(disc)
    assert SC.last == {"hit": False, "cached": False}
    monkeypatch.setenv("ENS_SETUP_CACHE", str(tmp_path))
    monkeypatch.setenv("ENS_SETUP_CACHE_MIN_DOFS", str(10 ** 9))
    SC.host_mesh(disc)
    assert SC.last["cached"] is False and not any(tmp_path.iterdir())
