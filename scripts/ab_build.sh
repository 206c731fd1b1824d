# Build/sort-stage A/B on one B200 (run under gpurun): build/sort parity tests, a c5 bench line,
# and ncu durations + DRAM bytes of the build and sort kernels.  usage: bash scripts/ab_build.sh TAG
mkdir -p gpurun_out
T=$1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "build or sort or occupancy or worked" > gpurun_out/t_$T.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/t_$T.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/b_c5_$T.json 2> gpurun_out/b_c5_$T.err; echo c5 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --kernel-name regex:"k_bin|k_scatter|k_stable_small|k_sort_small" -c 4 --csv --log-file gpurun_out/l_$T.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu rc=$?
python - $T <<'PY'
import csv,io,json,sys
T=sys.argv[1]
d=json.loads(open(f"gpurun_out/b_c5_{T}.json").read().strip().splitlines()[-1]); print("c5", round(d["ms_per_step"],2), {k: round(v,2) for k,v in d["stage_ms"].items()})
txt=open(f"gpurun_out/l_{T}.csv").read(); i=txt.index('"ID"'); rows=list(csv.reader(io.StringIO(txt[i:])))
h=rows[0]; acc={}
for r in rows[1:]:
    if len(r)<len(h): continue
    x=dict(zip(h,r)); acc.setdefault(x["ID"]+" "+x["Kernel Name"][:16],{})[x["Metric Name"]]=float(x["Metric Value"].replace(",",""))
for k,v in acc.items(): print(k, "ms %.3f rd %.2f GB wr %.2f GB instr %.2e"%(v["gpu__time_duration.sum"]/1e6, v["dram__bytes_read.sum"]/1e9, v["dram__bytes_write.sum"]/1e9, v["smsp__inst_executed.sum"]))
PY
