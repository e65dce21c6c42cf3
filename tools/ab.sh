# A/B the C4 bench across library builds: bash tools/ab.sh LIB1 LIB2 ...
for L in "$@"; do
  VPM_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done
