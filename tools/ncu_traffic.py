"""Developer: per-kernel DRAM traffic table from an `ncu --set full` raw page (ncu -i X.ncu-rep --page raw --csv).
usage: ncu_traffic.py raw.csv [out.json]
Prints one row per captured launch (time, DRAM bytes read / written, DRAM % of peak, warps active, registers) and,
with out.json, writes the first captured launch of each kernel class that bench.py's roofline reads
(profiles/r02_traffic.json: kernels[class] = {dram_bytes_per_launch, ncu_dram_pct_of_peak, ...})."""
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
h, units, data = rows[0], rows[1], rows[2:]
SC = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "usecond": 1e-3,
      "msecond": 1.0, "nsecond": 1e-6, "second": 1e3}


def col(name, r):
    i = h.index(name)
    return float(r[i].replace(",", "")) * SC.get(units[i], 1.0)


# profile class of bench.py's kernel table <- kernel name (first match wins)
CLASSES = [("op_node", "k_op_node_sym"), ("op_cell", "k_op_cell<0"), ("op_cell_fused", "k_op_cell<2"), ("step2", "k_op_cell<1"),
           ("step34", "k_step34"), ("ilu_steps678", "k_ilu_apply2"), ("mdot", "k_mdot2"), ("maxpy", "k_dcgs_update"),
           ("vc_resid_u_l0", ", 3, 0>(SymGeo"), ("vc_post_u_l0", ", 2, 0>(SymGeo"), ("vc_dscale_u_l0", "k_dscale"),
           ("vc_p7", "k_p7<")]
out, seen = {}, set()
print(f"{'kernel':46s} {'ms':>8s} {'rd GB':>8s} {'wr GB':>8s} {'DRAM%':>6s} {'warps%':>6s} {'regs':>4s} {'grid':>8s}")
for r in data:
    nm = r[h.index("Kernel Name")].replace("void ", "")
    ms, rd, wr = col("gpu__time_duration.sum", r), col("dram__bytes_read.sum", r), col("dram__bytes_write.sum", r)
    pct = col("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", r) if "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed" in h else float("nan")
    wa = col("sm__warps_active.avg.pct_of_peak_sustained_active", r)
    rg = col("launch__registers_per_thread", r)
    print(f"{nm.split('(')[0][:46]:46s} {ms:8.3f} {rd / 1e9:8.3f} {wr / 1e9:8.3f} {pct:6.1f} {wa:6.1f} {rg:4.0f} {col('launch__grid_size', r):8.0f}")
    for cls, key in CLASSES:
        if key in nm and cls not in seen:
            seen.add(cls)
            out[cls] = dict(kernel=nm.split("(")[0], dram_bytes_per_launch=rd + wr, dram_read=rd, dram_write=wr, ncu_ms=ms,
                            ncu_dram_pct_of_peak=pct, warps_active_pct=wa, registers=rg)
            break
if len(sys.argv) > 2:
    json.dump(dict(source=f"ncu --set full --clock-control none (tools/ncu_capture.sh), raw page {sys.argv[1]}; first captured "
                          "launch of each kernel (tools/ncu_traffic.py)",
                   note="traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch (cold cache, serialised)", kernels=out),
              open(sys.argv[2], "w"), indent=1)
