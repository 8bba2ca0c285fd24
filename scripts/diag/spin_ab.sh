# intra-CTA ring back-off A/B (diagnostics): TWB_SPIN_NS 128 (main) vs 32 vs 0
V=paper_2007_16135_b200/lib/variants
for rep in 1 2; do
for L in main spin32 spin0; do
  if [ $L = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$V/libtwb200_$L.so; fi
  echo "== $L rep $rep"
  python scripts/tune.py pair 100000 1 f64
  python scripts/tune.py pair 300000 1 f64
  python scripts/tune.py pair 300000 3 f64
  python scripts/tune.py pair 100000 3 f64
done; done
