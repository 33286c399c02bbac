timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for tc in 1 0; do
  ZKL_MV_TC=$tc ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_mvt_|k_mvw_rows|k_mvf_cols" --csv --log-file gpurun_out/mvt_tc$tc.csv python scratch/mv_bench.py > /dev/null 2>&1
done
python - <<'PY'
import csv, collections
for tc in (1, 0):
    rows = [r for r in csv.reader(open('gpurun_out/mvt_tc%d.csv' % tc)) if len(r) > 10]
    hdr = rows[0]; per = collections.defaultdict(dict)
    for r in rows[1:]: per[r[hdr.index("ID")]][r[hdr.index("Metric Name")]] = float(r[hdr.index("Metric Value")]); per[r[hdr.index("ID")]]["k"] = r[hdr.index("Kernel Name")][:30]
    grp = collections.defaultdict(list)
    for m in per.values(): grp[(m["k"], round(m["dram__bytes_read.sum"] / 1e6))].append(m["gpu__time_duration.sum"])
    print("TC=%d" % tc, {k: round(sum(v)/len(v)/1000, 1) for k, v in grp.items()})
PY
