timeout 120 python scripts/tune.py batch 2000 28 28 f64 1
timeout 120 python scripts/tune.py batch 2000 28 28 f32 1
timeout 120 python scripts/tune.py batch 1000 128 8 f64 0
timeout 200 python scripts/tune.py pair 100000 8 f64 0
timeout 200 python scripts/tune.py pair 100000 28 f64 0
