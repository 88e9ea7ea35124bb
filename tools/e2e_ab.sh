# e2e step times of library variants (TMOTIF_LIB), bench.py's e2e pass only
for lib in "$@"; do
  if [ "$lib" = base ]; then unset TMOTIF_LIB; else export TMOTIF_LIB=$lib; fi
  python bench.py --no-parity --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 8 2>&1 >/dev/null | grep "e2e steps" | sed "s|^|$lib |"
done
