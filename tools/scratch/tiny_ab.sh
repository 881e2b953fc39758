# tiny-kernel launches (latency and mid sizes) under the library builds in $LIBS
for i in 1 2; do for lib in $LIBS; do
  echo "== $lib"
  MPXA_LIB=ab/libmpxa_$lib.so SIZES_MIB=1,2 timeout 100 python tools/ag_tail.py
  MPXA_LIB=ab/libmpxa_$lib.so ALGOS=pairwise SIZES=16,4096,262144,524288 timeout 100 python tools/lat_knobs.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:v for k,v in d['us'].items() if not k.endswith('path')})"
done; done
