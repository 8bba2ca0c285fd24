# unroll of the rows-in-registers builds (diagnostics): 4 (main), 8, 16
V=paper_2007_16135_b200/lib/variants
for rep in 1; do
for L in ur8 ur16; do
  export TWB_LIBRARY=$V/libtwb200_$L.so
  echo "== $L rep $rep"
  python scripts/tune.py pair 100000 1 f64
  python scripts/tune.py pair 1000000 1 f64
  python scripts/tune.py pair 1000000 3 f32
  python scripts/tune.py pair 300000 1 f64
done; done
