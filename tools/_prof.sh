mkdir -p gpurun_out
export B200LU_BATCH_UNIT=16 B200LU_BATCH_SLOT_KB=1 B200LU_BATCH_RING_KB=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_batch.csv python tools/batch_probe.py C2 256 2 > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/launches_batch.csv")) if len(r)>5]
hdr=rows[0]; ik=hdr.index("Kernel Name"); iv=hdr.index("Metric Value")
for r in rows[1:]:
    if "btri" in r[ik] or "bfactor" in r[ik] or "bpermute" in r[ik]: print(r[ik][:60], r[iv])
PY
