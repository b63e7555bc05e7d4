"""Markdown rows of the stage-emulation table from emulate_stage.py outputs.

    python tools/emulation_table.py "label" file.json ["label" file.json ...]
"""
import json
import sys


def main():
    args = sys.argv[1:]
    print("| config (ledger budget) | stage | HEU | exposed span / overlapped | cross-check T(HEU)−T(elided) | elided "
          "| full recompute | selective (fits budget?) | simulator / measured |")
    print("|---|---|---|---|---|---|---|---|---|")
    for label, path in zip(args[::2], args[1::2]):
        d = json.load(open(path))
        first = True
        for s, row in sorted(d["stages"].items(), key=lambda kv: int(kv[0])):
            h, el = row["heu"], row["elided"]
            full, sel = row.get("full_recompute"), row.get("selective")
            selc = "—" if not sel else f"{sel['iteration_ms']:.0f} ({'yes' if sel.get('fits_budget') else 'no'})"
            print(f"| {label if first else ''} | {s} | {h['iteration_ms']:.0f} | {h['exposed_recompute_ms']:.1f} / "
                  f"{h['recompute_overlapped_ms']:.1f} | {row['crosscheck_ms']:.1f} | {el['iteration_ms']:.0f} | "
                  f"{full['iteration_ms']:.0f} | {selc} | {row['simulated_over_measured']:.3f} |"
                  if full else
                  f"| {label if first else ''} | {s} | {h['iteration_ms']:.0f} | {h['exposed_recompute_ms']:.1f} / "
                  f"{h['recompute_overlapped_ms']:.1f} | {row['crosscheck_ms']:.1f} | {el['iteration_ms']:.0f} | — | {selc} "
                  f"| {row['simulated_over_measured']:.3f} |")
            first = False


if __name__ == "__main__":
    main()
