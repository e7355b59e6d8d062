"""Binary store of a built Connectivity (one .npy per array + a small pickle).

Setup-side companion of the native builder: a connectivity built once (the
40M-point cloud takes ~90 s on 16 cores) is written to a directory and read
back memory-mapped, so the ranks of a multi-GPU run on one node share one
copy of the global stencil in the page cache (/dev/shm) instead of each
building and holding its own (8 x ~40 GB).  Split families are stored as
their sums and counts only (builder.SplitView derives the CSR on demand).
"""

from __future__ import annotations

import pickle
from pathlib import Path

import numpy as np

from . import geometry as G
from .builder import SplitView

_FULL = ("ptr", "idx", "dx", "dy", "sxx", "sxy", "syy", "det")
_CLOUD = ("x", "y", "flag", "nx", "ny")


def save(conn: G.Connectivity, path, extra: dict | None = None) -> None:
    d = Path(path)
    d.mkdir(parents=True, exist_ok=True)
    for k in _CLOUD:
        np.save(d / f"cloud_{k}.npy", getattr(conn.cloud, k))
    for k in _FULL:
        np.save(d / f"full_{k}.npy", getattr(conn.full, k))
    for f, kind in enumerate(G.SPLIT_KINDS):
        s = conn.split[kind]
        for k in ("sxx", "sxy", "syy", "det"):
            np.save(d / f"split{f}_{k}.npy", getattr(s, k))
        np.save(d / f"split{f}_counts.npy", np.asarray(s.counts()))
        np.save(d / f"det_safe{f}.npy", conn.det_safe[kind])
    np.save(d / "d_min.npy", conn.d_min)
    np.save(d / "d_mean.npy", conn.d_mean)
    for k, v in (extra or {}).items():
        np.save(d / f"extra_{k}.npy", v)
    with open(d / "frames.pkl", "wb") as fh:
        pickle.dump({"wall": conn.wall_frame, "outer": conn.outer_frame}, fh)
    (d / "DONE").write_text("ok")


def load(path, mmap: bool = True):
    """(Connectivity, extra arrays) from `save`; arrays memory-mapped."""
    d = Path(path)
    if not (d / "DONE").exists():
        raise FileNotFoundError(f"{d}: no complete connectivity store")
    mode = "r" if mmap else None
    ld = lambda name: np.load(d / name, mmap_mode=mode)  # noqa: E731
    cloud = G.PointCloud(*(np.asarray(ld(f"cloud_{k}.npy")) for k in _CLOUD))
    full = G.StencilSet(**{k: ld(f"full_{k}.npy") for k in _FULL})
    split, det_safe = {}, {}
    for f, kind in enumerate(G.SPLIT_KINDS):
        split[kind] = SplitView(full, f, ld(f"split{f}_counts.npy"),
                                *(ld(f"split{f}_{k}.npy") for k in ("sxx", "sxy", "syy", "det")))
        det_safe[kind] = ld(f"det_safe{f}.npy")
    with open(d / "frames.pkl", "rb") as fh:
        fr = pickle.load(fh)
    conn = G.Connectivity(cloud=cloud, full=full, split=split, d_min=ld("d_min.npy"), d_mean=ld("d_mean.npy"),
                          wall_frame=fr["wall"], outer_frame=fr["outer"], det_safe=det_safe)
    extra = {p.name[6:-4]: np.load(p, mmap_mode=mode) for p in d.glob("extra_*.npy")}
    return conn, extra
