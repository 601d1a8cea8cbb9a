for s in default 1,128 1,256 2,128 2,256; do
  if [ "$s" = default ]; then unset RDX_GEMM_SHAPE; else export RDX_GEMM_SHAPE=$s; fi
  timeout 300 python bench.py --no-cpu --steps 10 --warmup 3 > /tmp/b.json 2>/dev/null
  python -c "
import json;d=json.load(open('/tmp/b.json'))
print('$s', 'ms',d['ms_per_step'], {k:v['us_per_step'] for k,v in d['breakdown_us_radix'].items() if k.startswith('gemm')})"
done
