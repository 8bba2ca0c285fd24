# warp-ring size A/B (diagnostics): TWB_ZRS_REG 512 (main) vs 256 for the
# rows-in-registers configurations (d = 1 fp64, fp32 mode)
V=paper_2007_16135_b200/lib/variants
for rep in 1 2; do
for L in main zreg256; do
  if [ $L = main ]; then unset TWB_LIBRARY; else export TWB_LIBRARY=$V/libtwb200_$L.so; fi
  echo "== $L rep $rep"
  python scripts/tune.py pair 1000000 3 f64
  python scripts/tune.py pair 1000000 3 f32
  python scripts/tune.py pair 1000000 1 f64
  python scripts/tune.py pair 300000 1 f64
  python scripts/tune.py pair 100000 1 f64
  python scripts/tune.py pair 100000 3 f32
done; done
