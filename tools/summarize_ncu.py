"""Selected raw metrics of an .ncu-rep, one block per launch (run where ncu is installed)."""
import csv, re, subprocess, sys

PAT = re.compile(r"^(gpu__time_duration\.sum|dram__bytes_read\.sum|dram__bytes_write\.sum|"
                 r"gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed|"
                 r"sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_active|"
                 r"sm__warps_active\.avg\.pct_of_peak_sustained_active|launch__registers_per_thread|"
                 r"launch__grid_size|launch__block_size|launch__shared_mem_per_block_dynamic|"
                 r"l1tex__m_xbar2l1tex_read_bytes\.sum|lts__t_sector_hit_rate\.pct|"
                 r"sm__throughput\.avg\.pct_of_peak_sustained_elapsed|sm__cycles_elapsed\.max|"
                 r"sm__icc_request_hit_rate\.pct|smsp__inst_executed\.sum|"
                 r"smsp__issue_active\.avg\.pct_of_peak_sustained_active|"
                 r"smsp__average_warps_issue_stalled_(barrier|no_instruction|long_scoreboard|"
                 r"short_scoreboard|wait|membar|branch_resolving)_per_issue_active\.ratio)$")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"# {rep}")
    for r in rows[2:]:
        print("----")
        print("  Kernel Name =", r[hdr.index("Kernel Name")])
        for h, u, v in zip(hdr, units, r):
            if PAT.match(h):
                print(f"  {h} = {v} {u}")
