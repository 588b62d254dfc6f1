"""Dataset directories (fem.py:413-478) against a directory written by the
reference itself (tests/golden/make_dataset_golden.py): load, round-trip
byte-identically, split, and stack into a batch."""
import filecmp
import json
import os

import numpy as np
import pytest

from paper_2305_16432_b200 import datasets
from paper_2305_16432_b200.errors import DataFormatError, DimensionMismatchError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "dataset_heat_small")


def test_load_reference_dataset():
    manifest, trajs = datasets.load_dataset(GOLD)
    assert manifest["schema_version"] == 1 and manifest["kind"] == "heat"
    assert [t.meta["split"] for t in trajs] == ["train", "train", "test"]
    assert all(len(t) == 2 for t in trajs)
    tup = trajs[0].tuples[0]
    assert tup.A.n == tup.b.shape[0] == tup.x.shape[0]
    # the stored x solves the stored system (the reference solved to 1e-12)
    r = tup.b - tup.A.to_dense() @ tup.x
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(tup.b)
    assert len(datasets.split(trajs, "train")) == 4 and len(datasets.split(trajs, "test")) == 2


def test_roundtrip_is_byte_identical(tmp_path):
    manifest, trajs = datasets.load_dataset(GOLD)
    with open(os.path.join(GOLD, "mesh.obj"), encoding="ascii") as fh:
        obj = fh.read()
    datasets.save_dataset(tmp_path, manifest["config"], trajs, obj, manifest["name"], manifest["kind"],
                          manifest["seed"])
    names = sorted(os.listdir(GOLD))
    assert sorted(os.listdir(tmp_path)) == [n for n in names if not n.endswith(".py")]
    match, mismatch, errors = filecmp.cmpfiles(GOLD, tmp_path, names, shallow=False)
    assert not mismatch and not errors, (mismatch, errors)


def test_stack_tuples():
    _, trajs = datasets.load_dataset(GOLD)
    tuples = datasets.split(trajs, "train")
    groups = datasets.group_by_pattern(tuples)  # one Dirichlet set per trajectory
    assert [len(g) for g in groups] == [2, 2]
    A, values, rhs, x = datasets.stack_tuples(groups[1])
    assert values.shape == (A.nnz, 2) and rhs.shape == (A.n, 2) and x.shape == (A.n, 2)
    np.testing.assert_array_equal(values[:, 1], groups[1][1].A.values)
    with pytest.raises(DimensionMismatchError):
        datasets.stack_tuples(tuples)


def test_errors(tmp_path):
    with pytest.raises(DataFormatError):
        datasets.load_dataset(tmp_path)
    (tmp_path / "manifest.json").write_text(json.dumps({"schema_version": 2, "trajectories": []}))
    with pytest.raises(DataFormatError):
        datasets.load_dataset(tmp_path)
