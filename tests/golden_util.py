"""Loading the reference-produced golden vectors (tests/golden/*.npz)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["cfg1_trained", "cfg1_perturbed", "cfg2_small_f64", "cfg3_small_f64"]


class Golden:
    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(GOLDEN, name + ".npz"))
        self.z = {k: z[k] for k in z.files}
        self.meta = json.loads(str(self.z["meta"]))
        self.n = int(self.z["n"])
        self.row_ptr = self.z["row_ptr"]
        self.col_idx = self.z["col_idx"]
        self.values = self.z["values"]
        self.rhs = self.z["rhs"]

    def case(self, i):
        pre = f"c{i}_"
        return {k[len(pre):]: v for k, v in self.z.items() if k.startswith(pre)}

    @property
    def n_cases(self):
        return len({k.split("_")[0] for k in self.z if k.startswith("c") and k[1].isdigit()})

    def hyper_kwargs(self):
        m = self.meta
        if m["weights"] == "trained":
            return None
        return dict(l=1, h=m["h"], n_mp=m["n_mp"], l_mp=1, h_mp=m["h_mp"])

    def params(self):
        """Weights as a dict: the committed checkpoint, or create_model(seed)
        with processor output layers x10 (the recorded recipe)."""
        from oracle import port
        m = self.meta
        if m["weights"] == "trained":
            hp, params = port.load_checkpoint(os.path.join(GOLDEN, m["checkpoint"]))
            return hp, params
        hp = port.Hyper(width=m["width"], **self.hyper_kwargs())
        params = port.create_params(hp, m["seed"])
        for r in range(hp.n_mp):
            for s in ("node", "edge"):
                params[f"mp{r}.{s}.{hp.l_mp}.w"] = params[f"mp{r}.{s}.{hp.l_mp}.w"] * 10.0
        return hp, params

    def stored_params(self):
        return {k[len("param:"):]: v for k, v in self.z.items() if k.startswith("param:")}


def params_sha(params):
    import hashlib
    blob = np.concatenate([np.ravel(params[k]) for k in sorted(params)])
    return hashlib.sha256(blob.tobytes()).hexdigest()
