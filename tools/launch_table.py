#!/usr/bin/env python
"""Per-kernel table from an ncu launch list (tools only).

    python tools/launch_table.py gpurun_out/r02_launches.csv > table.md

Input: `ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...`.
Output: markdown rows `| launches | total ms | share | kernel |`, largest first,
then a total line.  Templates are kept, argument lists dropped.
"""
import csv
import sys
from collections import defaultdict


def main(path: str) -> int:
    rows = list(csv.reader(line for line in open(path) if line.startswith('"')))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v if unit in ("ms", "msecond") else v / 1e6
        name = r[ki]
        depth, cut = 0, len(name)
        for j, ch in enumerate(name):      # drop the argument list, keep template arguments
            if ch == "<":
                depth += 1
            elif ch == ">":
                depth -= 1
            elif ch == "(" and depth == 0:
                cut = j
                break
        name = name[:cut]
        tot[name] += ms
        cnt[name] += 1
    total = sum(tot.values())
    print("| launches | total ms | share | kernel |")
    print("|---|---|---|---|")
    for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {cnt[name]} | {ms:.3f} | {100 * ms / total:.2f} % | `{name[:120]}` |")
    print(f"\nTotal {total:.1f} ms over {sum(cnt.values())} launches.")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
