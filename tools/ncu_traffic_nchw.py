"""DRAM traffic of the NCHW-direct FP32 conv per layer (one ncu run per layer, second call):

    python tools/ncu_traffic_nchw.py profiles/r02_traffic_nchw_n128.json [batch]

Runs `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--clock-control none -k regex:conv_simt` on tools/run_nchw_layer.py for each of the 12 layers
and keeps the launches of the second call (the first warms up): the same DRAM counters an
`ncu --set full` capture reports, per conv call (a tail-split layer's two launches summed).
"""
import csv
import io
import json
import subprocess
import sys
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

dst = sys.argv[1]
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1}
layers = {}
for name in BENCHMARKS:
    r = subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
                        "--clock-control", "none", "-k", "regex:conv_simt", "--csv", sys.executable,
                        str(ROOT / "tools" / "run_nchw_layer.py"), name, str(batch)],
                       capture_output=True, text=True)
    rows = [x for x in csv.reader(io.StringIO(r.stdout)) if len(x) > 10]
    hdr = rows[0]
    ki, mi, ui, vi, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"),
                          hdr.index("Metric Value"), hdr.index("ID"))
    per = {}
    for x in rows[1:]:
        d = per.setdefault(int(x[ii]), {})
        u = x[ui]
        v = float(x[vi].replace(",", ""))
        d[x[mi]] = v * (tscale.get(u, 1) if x[mi] == "gpu__time_duration.sum" else scale.get(u, 1))
    ids = sorted(per)
    second = ids[len(ids) // 2:]  # two identical calls: the second half of the launches
    b = sum(per[i]["dram__bytes_read.sum"] + per[i]["dram__bytes_write.sum"] for i in second)
    t = sum(per[i]["gpu__time_duration.sum"] for i in second)
    cfg = replace(BENCHMARKS[name], batch=batch)
    layers[name] = {"conv_dram_bytes": b, "conv_algorithmic_bytes": cfg.conv_nchw_bytes(),
                    "ratio": b / cfg.conv_nchw_bytes(), "launches": len(second), "ncu_time_s": t}
    print(name, f"{b / 1e9:.3f} GB vs algorithmic {cfg.conv_nchw_bytes() / 1e9:.3f} GB", flush=True)
Path(dst).write_text(json.dumps({
    "capture": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
               "-k regex:conv_simt, tools/run_nchw_layer.py per layer (second call)",
    "batch": batch, "variant": "fp32-exact", "path": "nchw", "layers": layers}, indent=1))
