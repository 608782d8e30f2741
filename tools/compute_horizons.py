"""Write tests/golden/horizons.json: the oracle's forward-stable horizon k* of every committed
parity case (tests/horizons.py, reading R17).  Calls only gen/ and oracle/.

usage: python tools/compute_horizons.py [key-prefix ...]   (default: every case; merges into the file)
"""
import json
import os
import sys
import time

os.environ["OPENBLAS_NUM_THREADS"] = "1"      # as tests/conftest.py: host-independent oracle bits
os.environ["OPENBLAS_CORETYPE"] = "Haswell"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import horizons as H  # noqa: E402


def main(prefixes):
    data = {"horizons": {}, "run_to": {}}
    if os.path.exists(H.GOLDEN):
        with open(H.GOLDEN) as f:
            data = json.load(f)
    keys = [k for k in H.all_keys() if not prefixes or any(k.startswith(p) for p in prefixes)]
    for key in keys:
        t0 = time.time()
        p, spec, maxit, meth, mode = H._resolve(key, None)
        kstar, _ = H.stable_horizon(p, spec, maxit, meth, mode)
        data["horizons"][key] = kstar
        data["run_to"][key] = maxit
        print(f"{key}: k* = {kstar} of {maxit} ({time.time() - t0:.1f} s)", flush=True)
        data["thresh"] = H.THRESH
        data["written_by"] = "tools/compute_horizons.py (gen/ + oracle/ only)"
        with open(H.GOLDEN, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
