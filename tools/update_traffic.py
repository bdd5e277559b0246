"""profiles/traffic.json from a set of `ncu --set full` captures: tools/update_traffic.py <round tag> [workload]
reads gpurun_out/<tag>_<kernel>.ncu-rep, writes profiles/<tag>_<kernel>_summary.txt and the traffic entries bench.py reads."""
import csv, json, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
wl = sys.argv[2] if len(sys.argv) > 2 else "c3"
names = {"gicp_nn": "gicp_nn_kernel", "gicp_step": "gicp_step_kernel", "gicp_lin": "gicp_lin_kernel", "gicp_halve": "gicp_halve_kernel",
         "gicp_init": "gicp_init_kernel", "render_kernel": "render_kernel", "cost_kernel": "cost_kernel"}
tj = ROOT / "profiles" / "traffic.json"
db = json.loads(tj.read_text()) if tj.exists() else {}
db.setdefault(wl, {})
for short, full in names.items():
    rep = ROOT / "gpurun_out" / f"{tag}_{short}.ncu-rep"
    if not rep.exists():
        continue
    summ = ROOT / "profiles" / f"{tag}_{full}_summary.txt"
    summ.write_text(subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_top.py"), str(rep), "28"], capture_output=True, text=True).stdout)
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, r = rows[0], rows[1], rows[2]
    def val(name, scale_units=True):
        i = hdr.index(name)
        v = float(r[i].replace(",", ""))
        u = units[i]
        if scale_units:
            v *= {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(u, 1.0)
        return v
    db[wl][full] = {
        "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
        "duration_ms_under_ncu": val("gpu__time_duration.sum"),
        "source": f"profiles/{summ.name} (ncu --set full --clock-control none, " +
                  ("launch #9 of 30, " if short in ("gicp_nn", "gicp_step", "gicp_lin", "gicp_halve") else "") + f"{wl.upper()} 58,320 candidates)",
        "ncu": {"issue_slots_busy_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active", False),
                "fp64_pipe_pct": val("sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active", False),
                "dram_pct_of_peak": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", False),
                "l1tex_pct": val("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", False),
                "lanes_active_of_32": val("smsp__thread_inst_executed_per_inst_executed.ratio", False),
                "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active", False),
                "registers_per_thread": val("launch__registers_per_thread", False)}}
    print(full, db[wl][full]["dram_bytes_per_launch"] / 1e6, "MB", db[wl][full]["duration_ms_under_ncu"], "ms", db[wl][full]["ncu"])
tj.write_text(json.dumps(db, indent=1))
