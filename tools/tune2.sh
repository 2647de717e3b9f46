timeout 300 python -m pytest tests -m gpu -q --timeout 120 -x 2>&1 | grep -E "^(FAILED|ERROR)|passed|failed|Error" | head -10
echo "== C4-like 1000 rows f64 (cta)"
timeout 120 python tools/sweep_probe.py --obs 1000 --vars 50000 --sweeps 2 --variant cta --plans "1,32,32 1,16,64 1,8,128 1,4,256"
timeout 120 python tools/sweep_probe.py --obs 1000 --vars 50000 --sweeps 2 --variant cta --plans "1,32,32 1,16,64 1,8,128" --dtype f32
echo "== C4-like cluster 1000 rows"
timeout 120 python tools/sweep_probe.py --obs 1000 --vars 50000 --sweeps 2 --variant cluster --plans "2,16,32 4,8,32 2,8,64"
echo "== C2 4096 f64 cta/cluster"
timeout 120 python tools/sweep_probe.py --obs 4096 --vars 4096 --sweeps 2 --variant cta --plans "1,16,256 1,32,128"
timeout 120 python tools/sweep_probe.py --obs 4096 --vars 4096 --sweeps 2 --variant cluster --plans "4,32,32 8,16,32 16,8,32 4,8,128 8,4,128 16,2,128 4,16,64 8,8,64"
echo "== C1 10000 f64"
timeout 120 python tools/sweep_probe.py --obs 10000 --vars 100 --sweeps 20 --variant cluster --plans "16,32,32 16,8,96 16,4,160 8,8,160 16,16,64"
timeout 120 python tools/sweep_probe.py --obs 10000 --vars 100 --sweeps 20 --variant grid --plans "40,1,256 10,4,256"
echo "== grid 600k f64"
timeout 120 python tools/sweep_probe.py --obs 600000 --vars 64 --sweeps 2 --variant grid
timeout 120 python tools/sweep_probe.py --obs 1200000 --vars 64 --sweeps 2 --variant grid --dtype f32
