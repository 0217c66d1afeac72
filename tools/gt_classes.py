#!/usr/bin/env python3
"""Per-CTA-class timing of the fused kernel from a globaltimer trace (SF_DEBUG_SKIP=2048 debug
build; lines `SFGT bx by t_entry t_release t_exit t_eplanes t_transport`): median microseconds from griddep
release to e planes landed, to exit, and entry to exit, for interior / edge / corner CTAs.

    python tools/gt_classes.py gt.txt [grid_x grid_y]
"""
import statistics
import sys
from collections import defaultdict


def main():
    gx, gy = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (13, 11)
    rows = [tuple(int(x) for x in l.split()[1:]) for l in open(sys.argv[1]) if l.startswith("SFGT")]
    rows.sort(key=lambda r: r[2])
    n = gx * gy
    launches = [rows[i:i + n] for i in range(0, len(rows) - n + 1, n)][-10:]

    def cls(x, y):
        l, r, t, b = x == 0, x == gx - 1, y == 0, y == gy - 1
        if (l or r) and (t or b):
            return "corner"
        return "left" if l else "right" if r else "top" if t else "bottom" if b else "interior"

    d = defaultdict(lambda: defaultdict(list))
    for g in launches:
        for r in g:
            c = cls(r[0], r[1])
            d[c]["post"].append((r[4] - r[3]) / 1e3)
            d[c]["tot"].append((r[4] - r[2]) / 1e3)
            if len(r) > 5 and r[5]:
                d[c]["e"].append((r[5] - r[3]) / 1e3)
            if len(r) > 6 and r[6]:
                d[c]["tr"].append((r[6] - r[5]) / 1e3)
                d[c]["up"].append((r[4] - r[6]) / 1e3)
    print("| CTA class | CTAs | release -> e planes (us) | transport (us) | update + store (us) | release -> exit (us, median) | max | entry -> exit (us) |")
    print("|---|---|---|---|---|---|---|---|")
    for k in ["interior", "top", "bottom", "left", "right", "corner"]:
        v = d[k]
        if not v["post"]:
            continue
        e = f"{statistics.median(v['e']):.2f}" if v["e"] else "-"
        tr = f"{statistics.median(v['tr']):.2f}" if v["tr"] else "-"
        up = f"{statistics.median(v['up']):.2f}" if v["up"] else "-"
        print(f"| {k} | {len(v['post']) // len(launches)} | {e} | {tr} | {up} | {statistics.median(v['post']):.2f} | "
              f"{max(v['post']):.2f} | {statistics.median(v['tot']):.2f} |")


if __name__ == "__main__":
    main()
