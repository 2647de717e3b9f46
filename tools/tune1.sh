timeout 300 python -m pytest tests -m gpu -q --timeout 120 -x 2>&1 | grep -E "^(FAILED|ERROR)|passed|failed|Error" | head -10
echo "== C4-like 1000 rows f64 (cta)"
timeout 120 python tools/sweep_probe.py --obs 1000 --vars 50000 --sweeps 2 --variant cta --plans "1,4,256 1,8,128 1,2,512 1,16,64 1,32,32" 
echo "== C4-like cluster 1000 rows"
timeout 120 python tools/sweep_probe.py --obs 1000 --vars 50000 --sweeps 2 --variant cluster --plans "2,4,128 2,2,256 4,2,128 4,1,256"
echo "== C2 4096 f64 cta/cluster"
timeout 120 python tools/sweep_probe.py --obs 4096 --vars 4096 --sweeps 2 --variant cta --plans "1,16,256 1,8,512"
timeout 120 python tools/sweep_probe.py --obs 4096 --vars 4096 --sweeps 2 --variant cluster --plans "2,8,256 4,4,256 4,8,128 8,2,256 8,4,128 16,1,256 16,2,128"
echo "== C1 10000 f64"
timeout 120 python tools/sweep_probe.py --obs 10000 --vars 100 --sweeps 20 --variant cluster --plans "4,16,160 8,8,160 8,4,320 16,4,160 16,2,320 16,8,96"
timeout 120 python tools/sweep_probe.py --obs 10000 --vars 100 --sweeps 20 --variant grid --plans "40,1,256 20,2,256 10,4,256 5,8,256"
echo "== grid 600k f64"
timeout 120 python tools/sweep_probe.py --obs 600000 --vars 64 --sweeps 2 --variant grid
timeout 120 python tools/sweep_probe.py --obs 1200000 --vars 64 --sweeps 2 --variant grid --dtype f32
echo "== c5"
timeout 300 python bench.py --config c5 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-400
echo "== c4"
timeout 300 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-400
