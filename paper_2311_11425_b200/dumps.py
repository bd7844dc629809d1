"""Self-describing field dumps (run.dump_fields, run.py:202-211).

``dump_fields(prefix, mesh, state, t)`` writes ``prefix.bin`` (the raw
(nglobal, 5) float64 state, C order — byte-identical to the reference's
``ndarray.tofile``) and ``prefix.hdr`` (dims, variables, set, time, n_z,
columns); device states are copied to the host first.  ``load_fields`` reads
a dump back into a StateField (host).
"""

from __future__ import annotations

import numpy as np

from .state import StateField

__all__ = ["dump_fields", "load_fields"]


def dump_fields(path_prefix, mesh, state, t):
    arr = state.data
    if hasattr(arr, "cpu"):
        arr = arr.detach().cpu().numpy()
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    arr.tofile(path_prefix + ".bin")
    with open(path_prefix + ".hdr", "w") as f:
        f.write(f"dims {arr.shape[0]} {arr.shape[1]}\n")
        f.write("variables " + " ".join(state.variables) + "\n")
        f.write(f"set {state.set_name}\n")
        f.write(f"time {t:.17g}\n")
        f.write(f"n_z {mesh.n_z}\ncolumns {mesh.ncol}\n")


def load_fields(path_prefix):
    """(StateField, header dict) from a dump written by dump_fields (or the reference)."""
    hdr = {}
    with open(path_prefix + ".hdr") as f:
        for line in f:
            key, _, val = line.strip().partition(" ")
            hdr[key] = val
    ng, nv = (int(x) for x in hdr["dims"].split())
    data = np.fromfile(path_prefix + ".bin", dtype=np.float64).reshape(ng, nv)
    st = StateField(hdr["set"], data)
    if " ".join(st.variables) != hdr["variables"]:
        raise ValueError("dump variables do not match the equation set")
    hdr["time"] = float(hdr["time"])
    hdr["n_z"] = int(hdr["n_z"])
    hdr["columns"] = int(hdr["columns"])
    return st, hdr
