"""Summarise one `ncu --set full` capture (.ncu-rep) for profiles/: duration,
DRAM bytes per launch, throughput, pipe utilisation, occupancy and warp-stall
breakdown; optionally merge the DRAM traffic into profiles/ncu_traffic.json
(read by bench.py for the roofline's `traffic` field).

    python scripts/ncu_summary.py gpurun_out/full_r1c.ncu-rep [--traffic-json profiles/ncu_traffic.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor operand (smem) active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:] if len(r) == len(hdr)]


def num(d, u, k):
    v = d.get(k, "")
    try:
        return float(v.replace(",", "")) * UNIT.get(u.get(k, ""), 1.0)
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    traffic = {}
    if a.traffic_json and os.path.exists(a.traffic_json):
        traffic = json.load(open(a.traffic_json))
    for d, u in raw(a.rep):
        name = d.get("Kernel Name", "?")
        short = name.split("(")[0].replace("void ", "").replace("cgs::", "").split("<")[0]
        print(f"== {name[:110]}")
        for k, label in KEYS:
            v = d.get(k)
            if v is None:  # some sections prefix the metric name (e.g. "TPC.TriageCompute.")
                v = next((x for kk, x in d.items() if kk.endswith("." + k)), None)
            if v is None or v == "":
                continue
            print(f"  {label:24s} {v} {u.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    f = float(v)
                except ValueError:
                    continue
                if f >= 0.1:
                    stalls.append((f, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        print("  warp stalls per issued instruction: " + ", ".join(f"{n} {f:.2f}" for f, n in stalls))
        rd, wr = num(d, u, "dram__bytes_read.sum"), num(d, u, "dram__bytes_write.sum")
        dur = num(d, u, "gpu__time_duration.sum")
        if rd is not None and wr is not None:
            print(f"  DRAM traffic/launch     {(rd + wr) / 1e6:.2f} MB"
                  + (f"  ({(rd + wr) / dur / 1e9:.1f} GB/s over the launch)" if dur else ""))
            issue = num(d, u, "smsp__issue_active.avg.pct_of_peak_sustained_active")

            def metric(k):
                v = num(d, u, k)
                if v is None:
                    kk = next((x for x in d if x.endswith("." + k)), None)
                    v = num(d, u, kk) if kk else None
                return v
            # FP32 work: FADD + FMUL + 2 FFMA thread-instructions per elapsed cycle
            # (whole GPU) against 148 SMs x 128 lanes x 2 FLOP per cycle
            per = [metric(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
                   for op in ("fadd", "fmul", "ffma")]
            fp32 = (per[0] + per[1] + 2.0 * per[2]) if None not in per else None
            winst = metric("smsp__inst_executed.sum")
            tinst = metric("sass__thread_inst_executed_true_per_opcode")
            traffic[short] = {"bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                              "duration_s": dur, "issue_active_pct": issue,
                              "fma_pipe_pct": metric("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
                              "alu_pipe_pct": metric("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                              "xu_pipe_pct": metric("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                              "fp32_flop_per_cycle": fp32,
                              "fp32_frac_of_peak": fp32 / 37888.0 if fp32 is not None else None,
                              "lane_efficiency": tinst / (32.0 * winst) if winst and tinst else None,
                              "warp_instructions": winst,
                              "source": os.path.basename(a.rep)}
            t = traffic[short]
            if fp32 is not None:
                print(f"  FP32 FLOP/cycle         {fp32:.0f} of 37888 ({100 * t['fp32_frac_of_peak']:.1f}% of peak)")
            if t["lane_efficiency"]:
                print(f"  lane efficiency         {100 * t['lane_efficiency']:.1f}% (thread instr / 32 x warp instr)")
    if a.traffic_json:
        json.dump(traffic, open(a.traffic_json, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
