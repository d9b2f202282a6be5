"""Run bench.py over BASELINE configs (and optionally MAC-path ablations) on the GPU and collect the
JSON lines: python tools/sweep.py [--ablation] [--out profiles/r02_bench.json]."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = ["C4", "C1", "C2", "C3a", "C3b", "C5dw_4096", "C5dw_8192", "C5dw_16384", "C5pw_4096", "C5pw_8192",
           "C5pw_16384"]


def run(cfg, extra):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--steps", "20", "--warmup", "5",
           "--no-cpu-baseline"] + extra
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode or not lines:
        return {"config": cfg, "extra": extra, "error": (out.stderr or out.stdout)[-800:]}
    return json.loads(lines[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ablation", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_bench.json"))
    args = ap.parse_args()
    res = {}
    if args.ablation:
        for cfg in ("C2", "C3a", "C3b"):
            for path in ("default", "eager", "direct"):
                extra = [] if path == "default" else ["--mac-path", path]
                res[f"{cfg}/{path}"] = run(cfg, extra)
                r = res[f"{cfg}/{path}"]
                print(cfg, path, r.get("ms_per_step"), r.get("stages_ms"), flush=True)
    else:
        for cfg in CONFIGS:
            res[cfg] = run(cfg, [])
            r = res[cfg]
            print(cfg, r.get("value"), r.get("ms_per_step"), r.get("stages_ms"), flush=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
