"""Write the reference-format CSVs on the GPU: per-layer algorithms and the Fig. 4 ablation.

    python tools/report.py [batch] [outdir]
"""
import sys
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2306_14316_b200 import harness  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 128
outdir = Path(sys.argv[2]) if len(sys.argv) > 2 else Path("gpurun_out")
outdir.mkdir(exist_ok=True)
records, ablation = [], []
for cfg in harness.layer_configs(batch):
    for algo in ("im2win-opt", "im2win-basic", "im2win-fma", "im2win-tf32", "im2win-bf16", "cudnn", "im2col-cublas"):
        records.append(harness.run_bench(replace(cfg, algorithm=algo, repeats=3)))
        r = records[-1]
        print(f"{cfg.name:7s} {algo:14s} {r.tflops:8.2f} TF  peak_mem {r.peak_mem_bytes / 2**20:8.1f} MiB  {r.checksum}",
              flush=True)
        torch.cuda.empty_cache()
    ablation.extend(harness.run_ablation(replace(cfg, repeats=3)))
    print("  ablation", {r.variant: round(r.tflops, 2) for r in ablation[-4:]}, flush=True)
(outdir / f"layers_n{batch}.csv").write_text(harness.report_csv(records))
(outdir / f"ablation_n{batch}.csv").write_text(harness.report_csv(ablation))
