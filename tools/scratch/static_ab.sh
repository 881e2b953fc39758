# static-executor launches at mid sizes under the library builds in $LIBS
for i in 1 2; do for lib in $LIBS; do
  echo "== $lib"
  MPXA_LIB=ab/libmpxa_$lib.so P=32 SIZES_KIB=64 timeout 100 python tools/a2a_knobs.py
  MPXA_LIB=ab/libmpxa_$lib.so P=16 SIZES_KIB=256 timeout 100 python tools/a2a_knobs.py
  MPXA_LIB=ab/libmpxa_$lib.so ALGOS=bruck SIZES=1048576,4194304 timeout 100 python tools/lat_knobs.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:v for k,v in d['us'].items() if not k.endswith('path')})"
done; done
