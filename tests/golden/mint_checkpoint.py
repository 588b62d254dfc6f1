"""Mint the reference's trained HEAT_HYPER checkpoint (test-fixture generator).

Runs ONLY in the build container, where /root/reference is importable:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/mint_checkpoint.py tests/golden/heat_trained.json

This is exactly the reference acceptance recipe
(pkg/tests/conftest.py:61-98 -> fixtures.train_staged(create_model(HEAT_HYPER,
seed=7), heat_train), fixtures.py:115-133). The checkpoint is written with the
reference's own save_model (gnn.py:335-353), so it round-trips bitwise. The
committed JSON is the parity input; goldens reference the committed file, not
a re-mint (OpenBLAS kernel selection makes re-mints host dependent).
"""
import sys
import time

from pcgkit import gnn
from pcgkit.fem import generate_dataset, train_test_split
from pcgkit.fixtures import HEAT_HYPER, heat_dataset_config, train_staged


def main(out):
    train_tuples, _ = train_test_split(generate_dataset(heat_dataset_config()))
    t0 = time.perf_counter()
    model, hist = train_staged(gnn.create_model(HEAT_HYPER, seed=7), train_tuples)
    gnn.save_model(out, model)
    print(f"minted {out} in {time.perf_counter() - t0:.1f}s; final loss "
          f"{hist[-1] if hist else None}")


if __name__ == "__main__":
    main(sys.argv[1])
