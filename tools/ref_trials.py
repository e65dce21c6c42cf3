"""Run the UNMODIFIED reference executive (perchsim.nmpc.control_loop from
/root/reference, its own compiled stepping core from oracle/_ref) on the host, to
pin the GPU executive's trial statistics.  Container-only (reads /root/reference).

usage: python tools/ref_trials.py SEEDS MODES OUT.json     e.g. 0-9 all tests/golden/ref_trials.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import perchsim._accel as acc  # noqa: E402
from perchsim import nmpc  # noqa: E402
from perchsim.config import ExperimentConfig  # noqa: E402

from oracle import refcore  # noqa: E402

core = refcore.load()
assert core is not None, "build oracle/_ref first (oracle/build_ref.sh)"
acc._core, acc.HAVE_COMPILED, acc._active = core, True, "compiled"


def main():
    lo, hi = (int(v) for v in sys.argv[1].split("-"))
    modes = ["no_disturbance", "uncompensated", "compensated"] if sys.argv[2] == "all" else sys.argv[2].split(",")
    out = {"source": "perchsim.nmpc.control_loop (reference, compiled FP64 core), ExperimentConfig() defaults",
           "trials": {}}
    for mode in modes:
        for seed in range(lo, hi + 1):
            t0 = time.perf_counter()
            rec = nmpc.control_loop(ExperimentConfig(), mode, seed)
            out["trials"][f"{mode}/{seed}"] = {
                "final_error": rec.final_error, "steps": len(rec.times), "failure": rec.failure,
                "trigger_time": rec.trigger_time, "replans_accepted": sum(e.accepted for e in rec.replans),
                "replans": len(rec.replans), "final_state": rec.states[-1].tolist(),
                "seconds": time.perf_counter() - t0}
            print(mode, seed, out["trials"][f"{mode}/{seed}"], flush=True)
            with open(sys.argv[3], "w") as fh:
                json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
