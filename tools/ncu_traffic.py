"""DRAM traffic per launch from an `ncu --set full` capture of tools/run_all_layers.py.

    python tools/ncu_traffic.py gpurun_out/traffic.ncu-rep profiles/r01_traffic_n128.json [batch] [variant]

Launch order in the capture: for each layer, the transform kernel then the conv
kernel (the -k filter drops pack_filter).  Writes per-layer dram bytes next to
the algorithmic bytes (workloads.BenchConfig.transform_bytes / conv_bytes).
"""
import csv
import io
import json
import subprocess
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2306_14316_b200.workloads import BENCHMARKS  # noqa: E402

rep, dst = sys.argv[1], sys.argv[2]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 128
variant = sys.argv[4] if len(sys.argv) > 4 else "fp32-exact"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ki = hdr.index("Kernel Name")
rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
dur = hdr.index("gpu__time_duration.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1}


def val(r, i, table):
    return float(r[i].replace(",", "")) * table.get(units[i], 1)


launches = [(r[ki], val(r, rd, scale) + val(r, wr, scale), val(r, dur, tscale)) for r in data]
names = list(BENCHMARKS)
# group per layer: one transform launch, then one or two conv launches (the SIMT tail split)
groups = []
for k, b, t in launches:
    if "transform" in k:
        groups.append({"bt": b, "tt": t, "bc": 0.0, "tc": 0.0, "nc": 0})
    else:
        assert "conv_simt" in k and groups, k
        groups[-1]["bc"] += b
        groups[-1]["tc"] += t
        groups[-1]["nc"] += 1
assert len(groups) == len(names), f"expected {len(names)} layers, got {len(groups)}"
out = {"capture": "ncu --set full --clock-control none -k regex:'conv_simt|im2win_transform_pipe' "
                  f"python tools/run_all_layers.py --batch {batch} --variant {variant}",
       "batch": batch, "variant": variant, "layers": {}}
for name, g in zip(names, groups):
    cfg = replace(BENCHMARKS[name], batch=batch)
    out["layers"][name] = {"transform_dram_bytes": g["bt"], "transform_algorithmic_bytes": cfg.transform_bytes(),
                           "conv_dram_bytes": g["bc"], "conv_algorithmic_bytes": cfg.conv_bytes(),
                           "conv_launches": g["nc"], "transform_ncu_s": g["tt"], "conv_ncu_s": g["tc"]}
    print(f"{name:7s} transform {g['bt'] / 1e6:9.1f} MB (alg {cfg.transform_bytes() / 1e6:9.1f})  "
          f"conv {g['bc'] / 1e6:9.1f} MB (alg {cfg.conv_bytes() / 1e6:9.1f}) in {g['nc']} launch(es)")
Path(dst).write_text(json.dumps(out, indent=1) + "\n")
