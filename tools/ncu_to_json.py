#!/usr/bin/env python
"""Summarise an ncu capture (``ncu -i X.ncu-rep --page raw --csv`` output, or a
``--csv --log-file`` metrics list) into JSON: per kernel name, the mean of each
numeric metric over its launches (bytes, nanoseconds; raw-page units are
converted) and the launch count.

  python tools/ncu_to_json.py capture.csv [--prefix cfg2:c64:] > out.json
"""

from __future__ import annotations

import csv
import json
import sys
from collections import defaultdict


# raw-page units -> bytes / nanoseconds / Hz (launch lists are already in base units)
_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
          "ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9}


def _num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def short(name):
    """'void <unnamed>::m2l_rows_kernel<float, 4>(long, ...)' -> 'm2l_rows_kernel<float, 4>'"""
    depth, cut = 0, len(name)
    for i, ch in enumerate(name):
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            cut = i
            break
    return name[:cut].replace("void ", "").replace("<unnamed>::", "").strip()


def parse(path):
    rows = list(csv.reader(open(path, newline="")))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki = h.index("Kernel Name")
    out = defaultdict(lambda: defaultdict(list))
    if "Metric Name" in h:  # long format: one row per (launch, metric)
        mi, vi = h.index("Metric Name"), h.index("Metric Value")
        for r in rows[hdr + 1:]:
            if len(r) > vi and _num(r[vi]) is not None:
                out[short(r[ki])][r[mi]].append(_num(r[vi]))
    else:  # raw page: one row per launch, one column per metric (row 2 = units)
        units = rows[hdr + 1]
        for r in rows[hdr + 2:]:
            if len(r) != len(h):
                continue
            for j, name in enumerate(h):
                v = _num(r[j])
                if v is not None and "__" in name:
                    out[short(r[ki])][name].append(v * _SCALE.get(units[j].strip(), 1.0))
    res = {}
    for k, d in out.items():
        res[k] = {m: sum(v) / len(v) for m, v in d.items()}
        res[k]["launches"] = max(len(v) for v in d.values())
    return res


if __name__ == "__main__":
    prefix = sys.argv[sys.argv.index("--prefix") + 1] if "--prefix" in sys.argv else ""
    res = parse(sys.argv[1])
    json.dump({prefix + k: v for k, v in res.items()}, sys.stdout, indent=1, sort_keys=True)
    print()
