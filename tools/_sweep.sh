for cfg in "16 1 0 512" "32 1 0 512"; do set -- $cfg; echo "cfg $cfg"; B200LU_BATCH_UNIT=$1 B200LU_BATCH_SLOT_KB=$2 B200LU_BATCH_RING_KB=$3 B200LU_BATCH_CHAIN_WIDTH=$4 timeout 600 python tools/batch_probe.py C2 256 2 > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['runs'][-1]
  print(d['unit'], d['slot'], 'staged', d['staged_pairs_frac'], 'grid', d['grid'], 'factor', r['phases']['factor'], 'lower', r['phases']['lower'], 'upper', r['phases']['upper'], 'ok', d['lu_bitwise'], d['x_bitwise'], 'sys/s', d['systems_per_s'])
except Exception as e:
  print('FAILED', open('/tmp/o.txt').read()[-600:])"; done
