# Kernel-variant sweep on the C3 workload: prints linearize / evaluate kernel ms per variant.
run() {  # $1 = label, rest = env/args
  local label=$1; shift
  env "$@" python bench.py --profile --steps 20 --warmup 5 --no-cpu-baseline --no-lm --no-extra --no-c5 $BENCH_ARGS 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', 'lin %.3f ms' % d['ms_linearize_kernel'], 'eval %.3f ms' % d['ms_evaluate_kernel'], 'value %.0f' % d['value'])"
}
run default VGICP_LIB=$PWD/paper_2109_07073_b200/lib/libvgicp_b200.so
for v in paper_2109_07073_b200/lib_variants/*/; do [ -d "$v" ] || continue; v=${v%/}; run "$(basename $v)" VGICP_LIB=$PWD/$v/libvgicp_b200.so; done
