#!/bin/bash
# Round-2 measurement pass (run under gpurun from the repo root): GPU tests, smoke, bench (both arms, the driver's
# K/W), all-config sweep, ncu launch list of the bench command, ncu --set full of the bench kernel and the new ones.
TAG=${1:-r02h}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/rc.txt"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > "$OUT/nvsmi.txt" 2>&1
python -m paper_2111_00113_b200.build > "$OUT/build.log" 2>&1 || { echo "build failed"; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -rA > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/rc.txt"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
echo "bench-ref rc=$?" >> "$OUT/rc.txt"
timeout 900 python tools/sweep.py > "$OUT/sweep.jsonl" 2> "$OUT/sweep.err"; echo "sweep rc=$?" >> "$OUT/rc.txt"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_c3_bench.csv" \
  python bench.py --steps 1 --warmup 3 --no-oracle > "$OUT/ncu_launches.log" 2>&1; echo "ncu-list rc=$?" >> "$OUT/rc.txt"
python tools/launches.py "$OUT/launches_c3_bench.csv" > "$OUT/launches_summary_c3_bench.txt" 2>&1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:step3d_zmp --launch-skip 60 --launch-count 1 -o "$OUT/step3d_zmp_c3" -f \
  python tools/run_c3_once.py C3 1 > "$OUT/ncu_step.log" 2>&1; echo "ncu-step rc=$?" >> "$OUT/rc.txt"
timeout 900 $NCU -k regex:"assemble|sketch_v5" --launch-skip 2 --launch-count 2 -o "$OUT/assemble_sketch_c3" -f \
  python tools/run_c3_once.py C3 2 > "$OUT/ncu_asm.log" 2>&1; echo "ncu-asm rc=$?" >> "$OUT/rc.txt"
timeout 900 $NCU -k regex:block_cheb --launch-skip 3 --launch-count 1 -o "$OUT/block_cheb_c5b" -f \
  python tools/run_srr_once.py C5B 1 > "$OUT/ncu_block.log" 2>&1; echo "ncu-block rc=$?" >> "$OUT/rc.txt"
timeout 900 $NCU -k regex:srft_stage --launch-skip 6 --launch-count 2 -o "$OUT/srft_c3" -f \
  python tools/run_srft_once.py > "$OUT/ncu_srft.log" 2>&1; echo "ncu-srft rc=$?" >> "$OUT/rc.txt"
timeout 900 $NCU -k regex:hqr_kernel --launch-count 1 -o "$OUT/hqr_c5" -f \
  python tools/run_srr_once.py C5 1 > "$OUT/ncu_hqr.log" 2>&1; echo "ncu-hqr rc=$?" >> "$OUT/rc.txt"
timeout 900 $NCU -k regex:"csr_ell|csr_orth" --launch-skip 4 --launch-count 2 -o "$OUT/csr_c4" -f \
  python tools/run_cfg_once.py C4 > "$OUT/ncu_csr.log" 2>&1; echo "ncu-csr rc=$?" >> "$OUT/rc.txt"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_c4.csv" \
  python tools/run_cfg_once.py C4 > "$OUT/ncu_launches_c4.log" 2>&1
python tools/launches.py "$OUT/launches_c4.csv" > "$OUT/launches_summary_c4.txt" 2>&1
SKS_DEBUG_HQR=1 python tools/run_srr_once.py C5 2 > "$OUT/hqr_counters.txt" 2>&1
for r in "$OUT"/*.ncu-rep; do python tools/ncu_summary.py "$r"; done > "$OUT/ncu_summaries.txt" 2>&1
python - "$OUT" <<'PY'
import csv, io, subprocess, sys, json
out = sys.argv[1]
# DRAM traffic of the bench kernel per launch (for the bench line's roofline.traffic)
r = subprocess.run(["ncu", "-i", f"{out}/step3d_zmp_c3.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(r)))
if len(rows) > 2:
    d = dict(zip(rows[0], rows[2]))
    tr = float(d.get("dram__bytes_read.sum", "0").replace(",", "")) + float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
    u = dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * scale.get(u["dram__bytes_read.sum"], 1)
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * scale.get(u["dram__bytes_write.sum"], 1)
    json.dump({"C3": rd + wr, "source": f"{out}/step3d_zmp_c3.ncu-rep dram__bytes_read.sum + dram__bytes_write.sum"},
              open(f"{out}/step_traffic.json", "w"))
PY
cat "$OUT/rc.txt"
