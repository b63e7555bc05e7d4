"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of `bench.py`.

Takes the longest complete training step: the launches from an embedding forward that follows an
Adam launch through the next Adam launch. Writes the step's launches
(`--csv-out`, id,kernel,ns) and a per-kernel summary (`--json-out`).

    python tools/launch_summary.py gpurun_out/launches.csv --csv-out profiles/r01_launches_7b_step.csv \
        --json-out profiles/r01_launches_7b_step_summary.json --cmd "<the ncu command>"
"""
import argparse
import csv
import json
import re
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)  # drop the parameter list
    name = re.sub(r"^void ", "", name)
    return name.replace("lynx::<unnamed>::", "lynx::<unnamed>::")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launches")
    ap.add_argument("--csv-out", required=True)
    ap.add_argument("--json-out", required=True)
    ap.add_argument("--cmd", default="")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    rows = []
    with open(args.launches) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        rows.append((int(r["ID"]), short(r["Kernel Name"]), int(round(ns))))
    adam = [i for i, (_, k, _) in enumerate(rows) if "adam" in k]
    if len(adam) < 2:
        raise SystemExit("need two optimizer launches to delimit a step")
    # the complete steps (embedding forward after one optimizer launch through the next); the longest
    # one is the workload's (bench.py ends with a short tiny-config run)
    steps = []
    for a, b in zip(adam, adam[1:]):
        start = next((i for i in range(a + 1, b) if "embedding_fwd" in rows[i][1]), None)
        if start is not None:
            steps.append(rows[start:b + 1])
    step = max(steps, key=lambda st: sum(ns for _, _, ns in st))
    with open(args.csv_out, "w") as f:
        if args.cmd:
            f.write(f"# {args.cmd}\n")
        if args.note:
            f.write(f"# {args.note}\n")
        f.write("id,kernel,ns\n")
        for i, k, ns in step:
            f.write(f"{i},{k},{ns}\n")
    agg = defaultdict(lambda: [0, 0])
    for _, k, ns in step:
        agg[k][0] += 1
        agg[k][1] += ns
    total = sum(ns for _, _, ns in step)
    kernels = [{"kernel": k, "launches": n, "ms": round(ns / 1e6, 2), "share": round(ns / total, 4)}
               for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    with open(args.json_out, "w") as f:
        json.dump({"source": args.csv_out, "launches": len(step), "sum_ms": round(total / 1e6, 2),
                   "kernels": kernels}, f, indent=1)
    print(f"{len(step)} launches, {total / 1e6:.1f} ms")
    for k in kernels[:12]:
        print(f"  {k['share']:.3f} {k['ms']:9.2f} ms {k['launches']:5d}  {k['kernel']}")


if __name__ == "__main__":
    main()
