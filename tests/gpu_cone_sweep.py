"""Sweep of the cone-kernel decomposition (lanes per cone G, loads in flight per lane R, register-resident or
chunked) and of the -W'W scatter variants on the C4 cone layout.  Each configuration runs in a fresh process
(the knobs are read at handle creation).  Not a pytest file.

    python tests/gpu_cone_sweep.py            # prints one line per configuration
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def run(env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "gpu_microbench.py"), "10000", "20", "250", "0", "10"],
                       env=e, capture_output=True, text=True)
    if r.returncode != 0:
        return None, r.stderr[-400:]
    return json.loads(r.stdout.strip().splitlines()[-1])["kernels"], ""


def main():
    names = None
    for env in ([{"QS_WTW_STREAM": "1"}, {"QS_WTW_PLAIN": "1"}, {}] +
                [{"QS_CONE_G": str(g), "QS_CONE_SINGLE": str(s)} for g in (8, 16, 32) for s in (0, 1)]):
        k, err = run(env)
        if k is None:
            print(env, "FAILED", err)
            continue
        if names is None:
            names = list(k)
            print("config | " + " | ".join(n.split("(")[0] for n in names) + "   (warm us / cold us)")
        print(json.dumps(env), "|", " | ".join(f"{k[n]['us']:.1f}/{k[n]['cold_us']:.1f}" for n in names), flush=True)


if __name__ == "__main__":
    main()
