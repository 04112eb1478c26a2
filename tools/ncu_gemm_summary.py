"""Summarise an `ncu --set full` capture of tools/prof_gemm.py (the twelve stage
GEMMs of one layer, bench.py's roofline set) into profiles/gemm_traffic.json
(bench.py's roofline.traffic) and a text table (dev tool).

    python tools/ncu_gemm_summary.py gpurun_out/gemm_full.ncu-rep "<source line>"
"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = ["qkv fwd EPI_BF16 2048x6144x2048", "proj fwd EPI_RESID 2048x2048x2048",
         "fc1 fwd EPI_BIAS_GELU 2048x8192x2048", "fc2 fwd EPI_RESID 2048x2048x8192",
         "fc2 dgrad EPI_GELU_BWD 2048x8192x2048", "fc1 dgrad 2048x2048x8192", "qkv dgrad 2048x2048x6144",
         "fc2 wgrad EPI_ACC_F32 2048x8192x2048", "fc1 wgrad EPI_ACC_F32 8192x2048x2048",
         "qkv wgrad EPI_ACC_F32 6144x2048x2048", "proj dgrad 2048x2048x2048",
         "proj wgrad EPI_ACC_F32 2048x2048x2048"]
# algorithmic bytes (MB, 1e6): A + B read once (bf16), C written once (bf16; f32 accumulate:
# read + write); the residual / pre-activation operand R of EPI_RESID / EPI_GELU_BWD read once
_S, _D, _F = 2048, 2048, 8192
_MB = lambda *elems: round(sum(elems) / 1e6, 1)
ALG_MB = [_MB(2 * _S * _D, 2 * 3 * _D * _D, 2 * _S * 3 * _D),              # qkv fwd
          _MB(2 * _S * _D, 2 * _D * _D, 2 * _S * _D, 2 * _S * _D),           # proj fwd + R
          _MB(2 * _S * _D, 2 * _F * _D, 2 * 2 * _S * _F),                    # fc1 fwd (pre + act)
          _MB(2 * _S * _F, 2 * _D * _F, 2 * _S * _D, 2 * _S * _D),           # fc2 fwd + R
          _MB(2 * _S * _D, 2 * _D * _F, 2 * _S * _F, 2 * _S * _F),           # fc2 dgrad (+ pre)
          _MB(2 * _S * _F, 2 * _F * _D, 2 * _S * _D),                        # fc1 dgrad
          _MB(2 * _S * 3 * _D, 2 * 3 * _D * _D, 2 * _S * _D),                # qkv dgrad
          _MB(2 * _S * _D, 2 * _S * _F, 8 * _D * _F),                        # fc2 wgrad f32 +=
          _MB(2 * _S * _F, 2 * _S * _D, 8 * _F * _D),                        # fc1 wgrad f32 +=
          _MB(2 * _S * 3 * _D, 2 * _S * _D, 8 * 3 * _D * _D),                # qkv wgrad f32 +=
          _MB(2 * _S * _D, 2 * _D * _D, 2 * _S * _D),                        # proj dgrad
          _MB(2 * _S * _D, 2 * _S * _D, 8 * _D * _D)]                        # proj wgrad f32 +=


def main(rep, source):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    col = {}
    for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"):
        hits = [i for i, x in enumerate(h) if x == k] or [i for i, x in enumerate(h) if x.endswith("." + k)]
        col[k] = hits[0]
    units = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h) and "gemm_bf16" in r[col["Kernel Name"]]]

    def val(r, k, to):
        v = float(r[col[k]].replace(",", ""))
        u = units[col[k]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
        return v * scale.get(u, 1) / to

    ks, lines = [], []
    for i, r in enumerate(data[:len(NAMES)]):
        rd, wr = val(r, "dram__bytes_read.sum", 1e6), val(r, "dram__bytes_write.sum", 1e6)
        us = val(r, "gpu__time_duration.sum", 1)
        l2 = float(r[col["lts__throughput.avg.pct_of_peak_sustained_elapsed"]])
        tp = float(r[col["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]])
        ks.append({"gemm": NAMES[i], "kernel": r[col["Kernel Name"]].split("(")[0], "dram_read_MB": round(rd, 2),
                   "dram_write_MB": round(wr, 2), "traffic_MB": round(rd + wr, 2), "algorithmic_MB": ALG_MB[i],
                   "l2_pct": round(l2, 1), "ncu_us": round(us, 2), "tensor_pipe_active_pct": round(tp, 1)})
        lines.append(f"{NAMES[i]:38s} {us:7.1f} us  tensor {tp:5.1f}%  L2 {l2:5.1f}%  dram rd {rd:6.1f} wr {wr:5.1f} MB")
    mean = sum(k["traffic_MB"] for k in ks) / len(ks) * 1e6
    doc = {"source": source, "traffic_bytes_per_launch_mean": int(mean),
           "algorithmic_bytes_per_launch_mean": int(sum(ALG_MB) / len(ALG_MB) * 1e6),
           "note": "traffic < algorithmic: outputs stay in L2 at kernel end and operand re-reads are L2 hits",
           "kernels": ks}
    with open(os.path.join(ROOT, "profiles", "gemm_traffic.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print(source)
    print("\n".join(lines))
    print(f"mean dram traffic MB/launch {mean / 1e6:.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
