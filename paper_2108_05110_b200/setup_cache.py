"""On-disk cache of the per-mesh host setup.

`engine.HostMesh` -- the multifrontal plan (`symbolic.analyse`: nested
dissection, symbolic factorisation, launch schedule) plus the operator and slot
maps in the engine's internal numbering -- is a pure function of the
Discretization and of this package's code.  At BASELINE C5 it is ~13 s of the
~23 s setup on a 16-core host; the reference rebuilds its (smaller) setup every
run (`stepper.py:64-83`).  Here a mesh's HostMesh is written once to
``$ENS_SETUP_CACHE`` (default ``~/.cache/paper_2108_05110_b200``) as one .npy file
per array plus a JSON header, keyed by a SHA-256 of everything it depends on:

  * the mesh (vertices, triangles), both spaces' dof maps and coordinates, the
    pressure kind, the constrained rows / Dirichlet dofs / pin flag;
  * the operator values HostMesh copies (mass, stiffness, pressure integrals);
  * the source of the modules that compute it and the plan knobs (leaf size, panel
    width, split length).

A later run on the same mesh loads it (a few hundred ms per GB from the page
cache) instead of recomputing; any change to an input or to the code gives a new
key, and a missing, partial or unreadable entry just means a rebuild.  Only
meshes with at least ``ENS_SETUP_CACHE_MIN_DOFS`` (default 200 000) unknowns are
cached; ``ENS_SETUP_CACHE=off`` disables the cache.  Loaded arrays are
byte-identical to a fresh build (tests/test_setup_cache.py).  Timing runs
(bench.py) report the cold build and the warm load separately.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import shutil
import tempfile

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CODE = ("symbolic.py", "engine.py", "fe.py", "mesh.py", "discretization.py", "setup_cache.py",
         os.path.join("csrc", "host_symbolic.cpp"))
FORMAT = 1
last = {}          # what the last host_mesh() call did: {"hit": bool, "key": str, "load_s"/"save_s": float}


def cache_dir():
    d = os.environ.get("ENS_SETUP_CACHE", "")
    if d.lower() == "off":
        return None
    return d or os.path.join(os.path.expanduser("~"), ".cache", "paper_2108_05110_b200")


def min_dofs():
    return int(os.environ.get("ENS_SETUP_CACHE_MIN_DOFS", "200000"))


def _code_digest():
    h = hashlib.sha256()
    for name in _CODE:
        with open(os.path.join(_HERE, name), "rb") as fh:
            h.update(name.encode() + b"\0" + fh.read())
    return h.digest()


def mesh_key(disc) -> str:
    """SHA-256 over every input of HostMesh(disc) (module docstring)."""
    from . import symbolic as S
    h = hashlib.sha256()
    h.update(b"ensmhd-b200-hostmesh\0%d\0" % FORMAT)
    h.update(_code_digest())
    h.update(repr((S.LEAF_NODES, S.AMALGAMATE, S.PW, S.SPLIT_K, disc.pressure.kind, bool(disc.pin_pressure),
                   disc.n_scalar, disc.n_pres)).encode())

    def arr(a):
        a = np.ascontiguousarray(a)
        h.update(repr((a.dtype.str, a.shape)).encode())
        h.update(memoryview(a).cast("B"))

    vel, pres = disc.velocity, disc.pressure
    for a in (disc.mesh.vertices, disc.mesh.triangles, vel.cell_dofs, vel.dof_coords, pres.cell_dofs,
              pres.dof_coords, disc.constrained_rows, disc.bdofs, disc.pressure_integrals):
        arr(a)
    for m in (disc.mass_s, disc.stiff_s):
        arr(m.indptr)
        arr(m.indices)
        arr(m.data)
    return h.hexdigest()


def _scalar(v):
    return v.item() if isinstance(v, np.generic) else v


def _split(hm):
    """(meta, arrays) of a HostMesh: scalars into the JSON header, ndarrays into files."""
    meta = {"hm": {}, "plan": {}, "schedule": {}, "stats": {k: _scalar(v) for k, v in hm.plan.stats.items()}}
    arrays = {}
    for k, v in vars(hm).items():
        if k in ("disc", "plan") or v is None:
            continue
        if isinstance(v, np.ndarray):
            arrays["hm." + k] = v
        else:
            meta["hm"][k] = _scalar(v)
    for f in dataclasses.fields(hm.plan):
        v = getattr(hm.plan, f.name)
        if f.name in ("schedule", "stats"):
            continue
        if isinstance(v, np.ndarray):
            arrays["plan." + f.name] = v
        else:
            meta["plan"][f.name] = _scalar(v)
    for k, v in hm.plan.schedule.items():
        if isinstance(v, np.ndarray):
            arrays["schedule." + k] = v
        else:
            meta["schedule"][k] = _scalar(v)
    return meta, arrays


def save(hm, key):
    root = cache_dir()
    if root is None:
        return
    os.makedirs(root, exist_ok=True)
    final = os.path.join(root, key)
    if os.path.isdir(final):
        return
    tmp = tempfile.mkdtemp(prefix=key[:16] + ".", dir=root)
    try:
        meta, arrays = _split(hm)
        for name, a in arrays.items():
            np.save(os.path.join(tmp, name + ".npy"), a, allow_pickle=False)
        meta["arrays"] = sorted(arrays)
        with open(os.path.join(tmp, "meta.json"), "w") as fh:
            json.dump(meta, fh)
        os.replace(tmp, final)          # atomic publish: readers see a complete entry or none
    except (OSError, TypeError, ValueError):
        shutil.rmtree(tmp, ignore_errors=True)


def load(disc, key):
    """The cached HostMesh of ``disc``, or None."""
    from .engine import HostMesh
    from .symbolic import FactorPlan
    root = cache_dir()
    if root is None:
        return None
    d = os.path.join(root, key)
    try:
        with open(os.path.join(d, "meta.json")) as fh:
            meta = json.load(fh)
        arrays = {}
        for name in meta["arrays"]:
            arrays[name] = np.load(os.path.join(d, name + ".npy"), allow_pickle=False)
    except (OSError, ValueError, KeyError):
        return None
    hm = HostMesh.__new__(HostMesh)
    hm.disc = disc
    for k, v in meta["hm"].items():
        setattr(hm, k, v)
    fields = dict(meta["plan"])
    sched = dict(meta["schedule"])
    for name, a in arrays.items():
        grp, k = name.split(".", 1)
        if grp == "hm":
            setattr(hm, k, a)
        elif grp == "plan":
            fields[k] = a
        else:
            sched[k] = a
    hm.plan = FactorPlan(**fields, schedule=sched, stats=meta["stats"])
    hm._allkey = None
    return hm


def host_mesh(disc):
    """HostMesh(disc), through the on-disk cache for large meshes."""
    import time
    from .engine import HostMesh
    last.clear()
    if cache_dir() is None or disc.n_total < min_dofs():
        last.update(hit=False, cached=False)
        return HostMesh(disc)
    t = time.perf_counter()
    key = mesh_key(disc)
    last.update(key=key, key_s=time.perf_counter() - t)
    t = time.perf_counter()
    hm = load(disc, key)
    if hm is not None:
        last.update(hit=True, cached=True, load_s=time.perf_counter() - t)
        return hm
    hm = HostMesh(disc)
    t = time.perf_counter()
    save(hm, key)
    last.update(hit=False, cached=True, save_s=time.perf_counter() - t)
    return hm
