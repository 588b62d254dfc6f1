"""Mint a small dataset directory with the REFERENCE (pcgkit.fem.generate_dataset,
fem.py:381-400 + save_dataset fem.py:417-448) for tests/test_datasets.py.
Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_dataset_golden.py
"""
import os
import shutil

from pcgkit import fem

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "dataset_heat_small")

cfg = fem.DatasetConfig(name="heat-small", kind="heat", mesh_spec={"shape": "square", "k": 6},
                        n_trajectories=3, steps=2, seed=7, n_test_trajectories=1, dt=5e-2)
if os.path.exists(OUT):
    shutil.rmtree(OUT)
fem.generate_dataset(cfg, OUT)
print("wrote", OUT, sorted(os.listdir(OUT))[:6], "...")
