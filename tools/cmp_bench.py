"""Compare the us-per-call entries of bench.py JSON lines: python tools/cmp_bench.py A.json B.json ...
Prints entries whose best-of time differs by more than THRESH (default 8 %) between the first
half of the files (A) and the second half (B), each side taking the min over its files."""
import json, os, sys

THRESH = float(os.environ.get("THRESH", "0.08"))


def flat(x, path, out):
    if isinstance(x, dict):
        for k, v in x.items():
            flat(v, f"{path}/{k}", out)
    elif isinstance(x, list):
        if len(x) >= 2 and all(isinstance(v, (int, float)) for v in x[:2]) and not isinstance(x[0], bool):
            out[f"{path}[{x[0]}]"] = x[1]
        else:
            for i, v in enumerate(x):
                flat(v, f"{path}[{i}]", out)
    elif isinstance(x, (int, float)) and not isinstance(x, bool) and path.endswith("/us"):
        out[path] = x


def load(f):
    out = {}
    flat(json.loads(open(f).read().strip().splitlines()[-1]), "", out)
    return out


fs = sys.argv[1:]
h = len(fs) // 2
A = [load(f) for f in fs[:h]]
B = [load(f) for f in fs[h:]]
for k in A[0]:
    a = min(d[k] for d in A if k in d)
    if not all(k in d for d in B):
        continue
    b = min(d[k] for d in B)
    if a and b and abs(a - b) / max(a, b) > THRESH:
        print(f"{k:70s} {a:10.2f} {b:10.2f}  {b / a:5.2f}x")
