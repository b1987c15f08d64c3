"""Shared-memory atomic and bank-conflict counters, issue utilisation and DRAM throughput
of the SRWCR passes from an `ncu --set full` report (the report must show
dram__throughput and the shared-memory atomic wavefronts and bank conflicts for pass 1,
and name the binding unit).  usage: python tools/ncu_smem.py REPORT VOXELS > out.json"""
import csv, io, json, subprocess, sys
rep, vox = sys.argv[1], float(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
units = dict(zip(h, rows[1]))
want = {
    "dram_throughput_pct": "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_bytes_per_s": "dram__bytes.sum.per_second",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "shared_atom_inst": "smsp__inst_executed_op_shared_atom.sum",
    "shared_atom_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "shared_atom_wavefronts_pct_peak": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum.pct_of_peak_sustained_elapsed",
    "shared_atom_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "shared_ld_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "shared_st_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "lsu_shared_wavefronts_pct_peak": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "duration": "gpu__time_duration.sum",
    "warp_inst": "smsp__inst_executed.sum",
}
out = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
    e = {}
    for k, m in want.items():
        if m in d:
            try:
                e[k] = float(d[m].replace(",", ""))
            except ValueError:
                continue
            if units.get(m):
                e[k + "_unit"] = units[m]
    if "shared_atom_inst" in e and e["shared_atom_inst"] > 0:
        e["wavefronts_per_atom_inst"] = e["shared_atom_wavefronts"] / e["shared_atom_inst"]
    if "warp_inst" in e:
        e["warp_inst_per_32_voxels"] = e["warp_inst"] / (vox / 32)
        e["shared_atom_inst_per_32_voxels"] = e.get("shared_atom_inst", 0) / (vox / 32)
    e["binding_unit"] = ("issue (instruction issue slots)" if e.get("issue_active_pct", 0) > 65 else
                         "latency (issue slots idle, no unit saturated)")
    out[name] = e
print(json.dumps(out, indent=1))
