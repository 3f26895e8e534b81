"""Summarise an ncu report (ncu -i ... --page raw --csv) into a short text file.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/xxx.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_red.sum", "sm__cycles_elapsed.avg.per_second",
]


EXTRA_PREFIXES = ("l1tex__data_pipe_lsu_wavefronts", "smsp__issue_active.avg.pct",
                  "sm__inst_executed_pipe_lsu", "smsp__warps_active.avg.per_cycle_active",
                  "l1tex__t_bytes_pipe_lsu_mem_global_op_ld", "lts__t_bytes.sum",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
                  "sm__pipe_fma_cycles_active", "sm__pipe_alu_cycles_active",
                  "local_load", "local_store", "l1tex__t_sectors_pipe_lsu_mem_local")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("---")
        for k in KEYS:
            if k in d:
                print(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
        for k in sorted(d):
            if k.startswith(EXTRA_PREFIXES) or any(p in k for p in ("_mem_local",)):
                if k not in KEYS and d[k] not in ("", "n/a"):
                    print(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
        # warp stall breakdown: stalls per issued instruction, largest first
        st = []
        for k in d:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(d[k].replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        if st:
            st.sort(reverse=True)
            print("stalls_per_issue = " + ", ".join(f"{n} {v:.2f}" for v, n in st if v >= 0.05))
        rd = d.get("dram__bytes_read.sum")
        if rd is not None:
            def tobytes(k):
                v = float(d[k].replace(",", ""))
                s = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)
                return v * s
            print(f"dram_bytes_per_launch = {tobytes('dram__bytes_read.sum') + tobytes('dram__bytes_write.sum'):.0f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
