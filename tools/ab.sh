for L in paper_2509_16079_b200/lib/libvpm_b200.so build_exp/libvpm_u4.so build_exp/libvpm_u8.so build_exp/libvpm_rev.so paper_2509_16079_b200/lib/libvpm_b200.so; do
  VPM_LIB=$L python bench.py --steps 10 --warmup 3 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$L', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done
