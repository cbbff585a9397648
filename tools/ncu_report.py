"""Print the key metrics of an `ncu --set full` report (one kernel) as a markdown table.

usage: python tools/ncu_report.py gpurun_out/prof.ncu-rep [algorithmic_bytes]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "TMA load bytes (L2->SM)"),
    ("l1tex__m_l1tex2xbar_write_bytes_mem_global_op_tma_st.sum", "TMA store bytes"),
    ("sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum.pct_of_peak_sustained_elapsed", "tcgen05 INT8 ops % of peak"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA sub-pipe active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/LSU throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(path, alg_bytes=None):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    idx = {h: i for i, h in enumerate(hdr)}
    print("| metric | value |\n|---|---|")
    out = {}
    for k, name in KEYS:
        if k in idx:
            v, u = vals[idx[k]], units[idx[k]]
            out[k] = (v, u)
            print(f"| {name} (`{k}`) | {v} {u} |")
    if alg_bytes and "dram__bytes_read.sum" in out:
        def gb(vu):
            v, u = vu
            v = float(v.replace(",", ""))
            return v * {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "Tbyte": 1e3}.get(u, 1)
        traffic = gb(out["dram__bytes_read.sum"]) + gb(out["dram__bytes_write.sum"])
        print(f"| traffic / algorithmic bytes | {traffic:.3f} / {float(alg_bytes) / 1e9:.3f} GB = "
              f"{traffic / (float(alg_bytes) / 1e9):.2f} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
