"""Runs tools/_build/dropin_e2e (the C++ drop-in on the reference's types) on a
BASELINE config with MCMI_COMPAT_TRACE / MCMI_STREAM_DEBUG phase traces.

    python tools/e2e_cpp_probe.py [config] [runs] [VAR=a,b]   (VAR=...: A/B of an env knob)
"""
import os
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import numpy as np

    import bench
    name = sys.argv[1] if len(sys.argv) > 1 else "c2_sym27_1p3m"
    runs = sys.argv[2] if len(sys.argv) > 2 else "3"
    b, over = bench.workload(name)
    d = tempfile.mkdtemp(prefix="mcmi_probe_")
    np.array([b.n], np.int64).tofile(os.path.join(d, "n.i64"))
    b.row_ptr.astype(np.int64).tofile(os.path.join(d, "row_ptr.i64"))
    b.col_idx.astype(np.int64).tofile(os.path.join(d, "col_idx.i64"))
    b.values.astype(np.float64).tofile(os.path.join(d, "values.f64"))
    cmd = [os.path.join(REPO, "tools", "_build", "dropin_e2e"), d, repr(over.get("epsilon", 0.0625)),
           repr(over.get("delta", 0.0625)), repr(over.get("alpha", 5.0)), str(over.get("master_seed", 0)), runs]
    if len(sys.argv) > 3:  # A/B: VAR=a,b alternated 3 times, no traces
        var, vals = sys.argv[3].split("=")
        for rep in range(3):
            for v in vals.split(","):
                r = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, **{var: v}))
                print(f"{var}={v}", r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:],
                      flush=True)
        return
    env = dict(os.environ, MCMI_COMPAT_TRACE="1", MCMI_STREAM_DEBUG="1")
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    print(r.stderr)
    print(r.stdout)


if __name__ == "__main__":
    main()
