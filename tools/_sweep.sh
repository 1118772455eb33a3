for cfg in "16 1" "16 2" "16 3" "16 4" "16 5" "32 1" "32 3" "32 4"; do set -- $cfg; echo "cfg $cfg"; B200LU_BATCH_UNIT=$1 B200LU_BATCH_VARIANT=$2 timeout 600 python tools/batch_probe.py C2 256 2 > /tmp/o.txt 2>&1; tail -1 /tmp/o.txt | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['runs'][-1]
  print(d['unit'], d['slot'], 'grid', d['grid'], 'factor', r['phases']['factor'], 'lower', r['phases']['lower'], 'upper', r['phases']['upper'], 'ok', d['lu_bitwise'], d['x_bitwise'], 'sys/s', d['systems_per_s'])
except Exception as e:
  print('FAILED', open('/tmp/o.txt').read()[-600:])"; done
