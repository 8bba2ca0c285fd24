# CHS 16 (main) vs 32 with the 8-step unroll of the rows-in-registers builds (diagnostics)
V=paper_2007_16135_b200/lib/variants
for L in main chs32; do
  if [ $L = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$V/libtwb200_$L.so; fi
  echo "== $L"
  python scripts/tune.py pair 100000 1 f64
  python scripts/tune.py pair 1000000 1 f64
  python scripts/tune.py pair 1000000 3 f32
  python scripts/tune.py pair 1000000 3 f64
  python scripts/tune.py pair 300000 3 f64
done
