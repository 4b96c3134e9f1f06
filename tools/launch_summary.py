"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
profiles/<name>.md: per-kernel launch count, mean us and share of the
library's kernel time (torch setup kernels are listed separately).
usage: python tools/launch_summary.py gpurun_out/X_launches.csv profiles/r1_X_launches [cmd]"""
import collections
import csv
import sys

OURS = ("tree_", "argmax_keys", "greedy_walk", "row_stats", "stochastic_walk", "compact_kv", "paged_", "attend_",
        "merge_", "philox", "target_dist", "mss_", "fixup", "accept", "draft_", "stochastic_", "lazy_walk",
        "clear_words", "tape_", "sharded_")


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "")


def main(src, out, cmd=""):
    rows = []
    with open(src) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000.0 if unit == "ns" else v * (1000.0 if unit == "ms" else 1.0)
        rows.append((short(r["Kernel Name"]), us))
    ours = collections.OrderedDict()
    other = collections.OrderedDict()
    for n, us in rows:
        d = ours if any(n.startswith(p) or p in n for p in OURS) else other
        d.setdefault(n, []).append(us)
    tot = sum(sum(v) for v in ours.values())
    md = [f"# ncu launch list: `{src}`", "", f"command: `{cmd}`" if cmd else "", "",
          "Per-launch times are cold-cache and serialised (ncu replays each launch); "
          "compare SHARES with bench.py's kernels_ms, not absolutes.", "",
          "| kernel (library) | launches | mean us | share of library time |", "|---|---|---|---|"]
    for n, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        md.append(f"| `{n}` | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f} % |")
    md += ["", "| other (torch input setup) | launches | mean us |", "|---|---|---|"]
    for n, v in other.items():
        md.append(f"| `{n[:80]}` | {len(v)} | {sum(v) / len(v):.2f} |")
    open(out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md[:20]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], " ".join(sys.argv[3:]))
