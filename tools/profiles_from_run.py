"""Turn one tools/measure_r02.sh run (gpurun_out/m_*) into the committed profile files:

  profiles/r02_bench/{render,ref,train,knn}.json   the bench lines
  profiles/r02_render_launches.csv                  ncu launch list (gpu__time_duration.sum)
  profiles/r02_render_kernels_ncu_full.csv          ncu --set full, raw page of the render kernels
  profiles/ncu_traffic.json                         DRAM bytes per launch of each bench stage
  profiles/r02_tables.md                            the tables of r02_summary.md

usage: python tools/profiles_from_run.py [gpurun_out]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
OUT = os.path.join(ROOT, "profiles")

# bench stage -> the kernel (name prefix) whose ncu capture it uses (the longest launch
# of that name: the human field's, not the object's)
STAGE_KERNEL = {
    "human_canon": "human_canon_kernel",
    "human_deform_mlp": "deform_mlp_prec_kernel",
    "human_color_mlp": "color_mlp_prec_kernel",
    "march": "march_kernel",
}


def bench_lines():
    os.makedirs(os.path.join(OUT, "r02_bench"), exist_ok=True)
    lines = {}
    for name, log in (("render", "m_render"), ("ref", "m_ref"), ("train", "m_train"), ("knn", "m_knn")):
        js = [ln for ln in open(os.path.join(SRC, log + ".log")) if ln.startswith("{")]
        d = json.loads(js[-1])
        lines[name] = d
        with open(os.path.join(OUT, "r02_bench", name + ".json"), "w") as f:
            json.dump(d, f, indent=1)
    return lines


def launches():
    raw = open(os.path.join(SRC, "m_render_launches.csv")).read().splitlines()
    body = [ln for ln in raw if ln.startswith('"')]
    with open(os.path.join(OUT, "r02_render_launches.csv"), "w") as f:
        f.write("\n".join(body) + "\n")
    rows = list(csv.DictReader(io.StringIO("\n".join(body))))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        k = k.split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        per[k][0] += 1
        per[k][1] += v / 1000.0 if unit == "ns" else v if unit == "us" else v * 1000.0
    return per


def ncu_full():
    rep = os.path.join(SRC, "m_render_full.ncu-rep")
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith('"')]
    with open(os.path.join(OUT, "r02_render_kernels_ncu_full.csv"), "w") as f:
        f.write("\n".join(lines) + "\n")
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {k: i for i, k in enumerate(hdr)}
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def g(r, k):  # time in us, bytes in bytes, the rest as printed
        try:
            return float(r[col[k]].replace(",", "")) * scale.get(units[col[k]], 1.0)
        except (KeyError, ValueError):
            return float("nan")
    kern = []
    for r in data:
        name = r[col["Kernel Name"]].replace("void ", "").replace("<unnamed>::", "").split("(")[0]
        kern.append(dict(name=name, us=g(r, "gpu__time_duration.sum"),
                         regs=g(r, "launch__registers_per_thread"),
                         warps=g(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
                         tensor=g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
                         if "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" in col else
                         g(r, "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"),
                         l1=g(r, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
                         rd=g(r, "dram__bytes_read.sum"), wr=g(r, "dram__bytes_write.sum")))
    return kern


def main():
    lines = bench_lines()
    per = launches()
    kern = ncu_full()
    traffic = {}
    for stage, kname in STAGE_KERNEL.items():
        hits = [k for k in kern if k["name"].startswith(kname)]
        if hits:
            k = max(hits, key=lambda h: h["us"])
            traffic["fp32:" + stage] = {
                "dram_bytes_per_launch": (k["rd"] + k["wr"]),
                "source": "profiles/r02_render_kernels_ncu_full.csv (dram__bytes_read.sum + dram__bytes_write.sum, "
                          "one ncu --set full launch)"}
    with open(os.path.join(OUT, "ncu_traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    md = ["## Bench lines", "", "| workload | device time | e2e | notes |", "|---|---|---|---|"]
    rd = lines["render"]
    md.append(f"| configs[1] 512² view, fp32 semantics | {rd['ms_per_step']:.3f} ms/frame, {rd['value'] / 1e9:.3f} G samples/s"
              f" | {rd['e2e']['ms_per_step']:.3f} ms, {rd['e2e']['value'] / 1e9:.3f} G samples/s | "
              f"{rd['gpu_launches_detail']['per_step']} kernels/frame, "
              f"{rd['gpu_launches_detail']['foreign_kernels_per_step']} foreign; fp16 mode "
              f"{rd['fp16_mode']['ms_per_step']:.3f} ms |")
    rf = lines["ref"]
    md.append(f"| `--impl reference` (CPU port, same frames) | {rf['ms_per_step'] / 1e3:.2f} s/frame, "
              f"{rf['value'] / 1e6:.2f} M samples/s | same | no repository library loaded |")
    tr = lines["train"]
    md.append(f"| configs[2] training step | {tr['ms_per_step']:.1f} ms, {tr['value'] / 1e6:.0f} M samples/s | "
              f"{tr['e2e']['ms_per_step']:.1f} ms (eager, host batches) | "
              f"{tr['gpu_launches_detail']['per_step'] if 'gpu_launches_detail' in tr else ''} kernels/step |")
    roof = rd["roofline"]
    md += ["", f"Render roofline (dominant kernel): `{roof.get('kernel', '')}` {roof['achieved']:.0f} {roof['unit']}"
               f" = {roof['frac']:.3f} of {roof['peak']}.", "All stages: " + ", ".join(
                   f"{k} {v['ms'] * 1e3:.1f} us {v['frac']:.3f} ({v['bound']})" for k, v in roof["all_stages"].items()),
           "", "## Render launch list (one bench run: warm-up + timed frames + setup)", "",
           "| kernel | launches | µs total | share |", "|---|---|---|---|"]
    tot = sum(v[1] for v in per.values())
    for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f} % |")
    md += ["", "## ncu --set full (render kernels)", "",
           "| kernel | µs | regs | warps active % | tensor pipe % | L1TEX % | DRAM read / write MB |",
           "|---|---|---|---|---|---|---|"]
    for k in kern:
        md.append(f"| `{k['name']}` | {k['us']:.1f} | {k['regs']:.0f} | {k['warps']:.1f} | {k['tensor']:.1f} | "
                  f"{k['l1']:.1f} | {k['rd'] / 1e6:.2f} / {k['wr'] / 1e6:.2f} |")
    with open(os.path.join(OUT, "r02_tables.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
