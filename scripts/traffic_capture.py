"""DRAM traffic of the bench's dominant kernel class from an ncu metrics capture
of scripts/one_step.py (warm-up step + measured step, same build):

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic.csv python scripts/one_step.py
  python scripts/traffic_capture.py gpurun_out/traffic.csv profiles/r2_traffic.json

Writes per-class totals of the measured (second) step plus the sha256 of the
libhodlrgp_b200.so that ran and of its sources, so bench.py only uses the
figure for the same build (dividing the class's step bytes by its own ledger call count).
"""
import collections
import csv
import hashlib
import json
import re
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2303_10102_b200", "lib", "libhodlrgp_b200.so")

# kernel -> ledger class (csrc/prof.cuh PROF_*; the ProfScope each kernel runs under)
CLASSES = {
    "seg_tn": ("k_seg_tn", "k_seg_reduce", "k_proj_cat", "k_cat_reduce", "k_leafid_proj", "k_leafid_fold",
               "k_ml_proj", "k_ml_reduce", "k_ml_update", "k_ml_update_packed"),
    "seg_nn": ("k_seg_nn", "k_seg_nn_stream"),
    "leaf_mm": ("k_leaf_mm", "k_leaf_mm_dot"),
    "matvec": ("k_mv_",),
}


def kernel_base(name):
    """'void unnamed>::k_seg_tn<80, 80>(unnamed>::SegTnArgs)' -> 'k_seg_tn' (every
    kernel of the library is named k_*)."""
    m = re.search(r"\b(k_[A-Za-z0-9_]+)", name)
    return m.group(1) if m else name


def klass(base):
    for c, names in CLASSES.items():
        if any(base == n or (n.endswith("_") and base.startswith(n)) for n in names):
            return c
    return "other:" + base


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ii], {"kernel": r[ki]})
        d[r[ni]] = float(r[vi].replace(",", ""))
    launches = list(per.values())
    step = launches[len(launches) // 2:]
    agg = collections.defaultdict(collections.Counter)
    for d in step:
        c = klass(kernel_base(d["kernel"]))
        agg[c]["kernels"] += 1
        agg[c]["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        agg[c]["ns"] += d.get("gpu__time_duration.sum", 0)
    sys.path.insert(0, ROOT)
    from paper_2303_10102_b200.hodlrgp import source_sha256

    out = {"lib_sha256": hashlib.sha256(open(LIB, "rb").read()).hexdigest(), "src_sha256": source_sha256(),
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none, second step of scripts/one_step.py",
           "step_kernels": len(step),
           "classes": {c: {"kernels": v["kernels"], "dram_bytes": v["bytes"], "ms_cold": v["ns"] / 1e6}
                       for c, v in sorted(agg.items(), key=lambda x: -x[1]["ns"])}}
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    for c, v in list(out["classes"].items())[:12]:
        print(f"{c:32s} kernels {v['kernels']:6d} dram {v['dram_bytes'] / 1e9:9.3f} GB  {v['ms_cold']:9.3f} ms")


if __name__ == "__main__":
    main()
