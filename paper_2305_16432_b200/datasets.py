"""Dataset directories (mirrors the persistence half of pcgkit.fem,
/root/reference/pkg/src/pcgkit/fem.py:413-478): ``manifest.json`` (schema
1) plus Matrix Market files per tuple, and the mesh as OBJ text.

``load_dataset`` reads directories written by pcgkit (or by
``save_dataset`` here) into the same (manifest, trajectories) shape;
``save_dataset`` writes the manifest byte-identically to pcgkit for the same
content. The solve-path addition is ``stack_tuples``: tuples that share one
sparsity pattern become one batched problem -- a pattern matrix, values
(nnz, B) and right-hand sides (n, B) -- ready for
``gnn.build_learned_batch`` / ``pcg.pcg_solve_batch``.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

from . import mmio
from .errors import DataFormatError, DimensionMismatchError
from .sparse import SparseMatrixCsr

SCHEMA_VERSION = 1


@dataclass(frozen=True)
class DatasetTuple:
    A: SparseMatrixCsr
    b: np.ndarray
    x: np.ndarray
    meta: dict


@dataclass(frozen=True)
class Trajectory:
    tuples: list
    meta: dict

    def __len__(self):
        return len(self.tuples)


def _tuple_id(traj_id: int, step: int) -> str:
    """fem.py:413-414"""
    return f"t{traj_id:03d}_s{step:03d}"


def save_dataset(out_dir, config: dict, trajectories, mesh_obj_text: str, name: str, kind: str,
                 seed: int) -> None:
    """fem.py:417-448 with the config given as its JSON dict (pcgkit's
    ``_config_as_json(cfg)``) and the mesh as OBJ text."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "mesh.obj"), "w", encoding="ascii", newline="\n") as fh:
        fh.write(mesh_obj_text)
    manifest = {"schema_version": SCHEMA_VERSION, "name": name, "kind": kind, "mesh_file": "mesh.obj",
                "seed": seed, "config": config, "trajectories": []}
    for traj in trajectories:
        traj_id = traj.meta["trajectory"]
        entry = {"id": traj_id, "split": traj.meta["split"],
                 "params": {k: v for k, v in traj.meta.items() if k not in ("trajectory", "split")},
                 "tuples": []}
        for tup in traj.tuples:
            tid = _tuple_id(traj_id, tup.meta["step"])
            files = {"A": f"A_{tid}.mtx", "b": f"b_{tid}.mtx", "x": f"x_{tid}.mtx"}
            mmio.save_matrix(os.path.join(out_dir, files["A"]), tup.A)
            mmio.save_vector(os.path.join(out_dir, files["b"]), tup.b)
            mmio.save_vector(os.path.join(out_dir, files["x"]), tup.x)
            entry["tuples"].append({"id": tid, "files": files, "meta": tup.meta})
        manifest["trajectories"].append(entry)
    with open(os.path.join(out_dir, "manifest.json"), "w", encoding="ascii", newline="\n") as fh:
        json.dump(manifest, fh, sort_keys=True, indent=1)
        fh.write("\n")


def load_dataset(path) -> tuple[dict, list]:
    """fem.py:457-478: (manifest, trajectories); DataFormatError for a
    missing / unreadable manifest or another schema version."""
    manifest_path = os.path.join(path, "manifest.json")
    try:
        with open(manifest_path, encoding="ascii") as fh:
            manifest = json.load(fh)
    except (OSError, json.JSONDecodeError) as exc:
        raise DataFormatError(f"cannot read manifest at {manifest_path}: {exc}") from exc
    if manifest.get("schema_version") != SCHEMA_VERSION:
        raise DataFormatError("unsupported dataset schema version")
    trajectories = []
    for entry in manifest["trajectories"]:
        tuples = []
        for rec in entry["tuples"]:
            files = rec["files"]
            A = mmio.load_matrix(os.path.join(path, files["A"]))
            b = mmio.load_vector(os.path.join(path, files["b"]))
            x = mmio.load_vector(os.path.join(path, files["x"]))
            tuples.append(DatasetTuple(A, b, x, rec["meta"]))
        meta = dict(entry["params"], trajectory=entry["id"], split=entry["split"])
        trajectories.append(Trajectory(tuples, meta))
    return manifest, trajectories


def split(trajectories, which: str) -> list:
    """fem.py:402-405: the tuples of the "train" or "test" trajectories."""
    return [t for traj in trajectories if traj.meta["split"] == which for t in traj.tuples]


def stack_tuples(tuples):
    """Tuples on one sparsity pattern -> (A (pattern, values of the first),
    values (nnz, B), rhs (n, B), x (n, B)); DimensionMismatchError when the
    patterns differ."""
    if not tuples:
        raise DimensionMismatchError("no tuples to stack")
    A0 = tuples[0].A
    for t in tuples[1:]:
        if t.A.n != A0.n or not (np.array_equal(t.A.row_ptr, A0.row_ptr) and np.array_equal(t.A.col_idx, A0.col_idx)):
            raise DimensionMismatchError("tuples do not share one sparsity pattern")
    values = np.stack([t.A.values for t in tuples], axis=1)
    rhs = np.stack([np.asarray(t.b, dtype=np.float64) for t in tuples], axis=1)
    x = np.stack([np.asarray(t.x, dtype=np.float64) for t in tuples], axis=1)
    return A0, np.ascontiguousarray(values), np.ascontiguousarray(rhs), np.ascontiguousarray(x)


def group_by_pattern(tuples) -> list:
    """Tuples partitioned by sparsity pattern (first-appearance order), each
    group ready for stack_tuples -- trajectories with different Dirichlet
    sets land in different groups."""
    groups, keys = [], []
    for t in tuples:
        key = (t.A.n, t.A.row_ptr.tobytes(), t.A.col_idx.tobytes())
        if key in keys:
            groups[keys.index(key)].append(t)
        else:
            keys.append(key)
            groups.append([t])
    return groups
