"""Summarise an ncu --set full report (raw page) into JSON + a short table.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_summary.json --config 512x512x512
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_pct_peak": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_per_sm": ("sm__warps_active.avg.per_cycle_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "warp_insts": ("smsp__inst_executed.sum", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6 * 1e6, "us": 1e3,
        "ms": 1e6, "msecond": 1e6, "usecond": 1e3, "nsecond": 1}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--config", default="512x512x512")
    ap.add_argument("--voxels", type=float, default=512.0 ** 3)
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = {"report": a.report, "config": a.config, "kernels": {}}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        key = ("xy" if ("xy_kernel" in name or "xy2_kernel" in name or "xy2_hh_kernel" in name) else
               "zst" if ("zst_kernel" in name or "zst4_kernel" in name) else name[:40])
        d = {}
        for k, (m, _) in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if k.startswith("dram_") and k != "dram_pct_peak":
                    v *= UNIT.get(u, 1.0)
                if k == "time_ms":
                    v = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                             "msecond": 1.0}.get(u, 1e-6)
                d[k] = v
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        d["dram_bytes_per_voxel"] = d["dram_bytes_per_launch"] / a.voxels
        d["thread_insts_per_voxel"] = d.get("warp_insts", 0) * 32 / a.voxels
        d["config"] = a.config
        d["name"] = name
        out["kernels"][key] = d
    json.dump(out, open(a.out, "w"), indent=1)
    for k, d in out["kernels"].items():
        print(f"{k:6s} {d.get('time_ms', 0):7.3f} ms  dram {d['dram_bytes_per_voxel']:6.2f} B/vox "
              f"({d.get('dram_pct_peak', 0):4.1f}% peak)  issue {d.get('issue_active_pct', 0):4.1f}%  "
              f"fma {d.get('fma_pipe_pct', 0):4.1f}%  warps/SM {d.get('warps_active_per_sm', 0):4.1f}  "
              f"regs {d.get('regs', 0):.0f}  insts/vox {d['thread_insts_per_voxel']:.0f}")


if __name__ == "__main__":
    main()
