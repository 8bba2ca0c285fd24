# steady-loop unroll A/B (diagnostics): TWB_WAVE_UNROLL 2 (main) vs 1 vs 4
V=paper_2007_16135_b200/lib/variants
for rep in 1 2; do
for L in main unr1 unr4; do
  if [ $L = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$V/libtwb200_$L.so; fi
  echo "== $L rep $rep"
  python scripts/tune.py pair 100000 1 f64
  python scripts/tune.py pair 1000000 1 f64
  python scripts/tune.py pair 1000000 3 f32
  python scripts/tune.py pair 1000000 3 f64
done; done
