# every BASELINE config through bench.py (one JSON line each) -> gpurun_out/bench_all.jsonl;
# C1 / C2 / C4 also with the labelled block-Gram sweep (--variant bgram)
mkdir -p gpurun_out
: > gpurun_out/bench_all.jsonl
for c in c1 c2 c2b c4 c5 c3f32 c3s8 c3 p1 p3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 ${BENCH_EXTRA} >> gpurun_out/bench_all.jsonl 2> gpurun_out/bench_$c.err || echo "{\"config\": \"$c\", \"failed\": true}" >> gpurun_out/bench_all.jsonl
done
for c in c1 c2 c4; do
  timeout 900 python bench.py --config $c --variant bgram --steps 3 --warmup 3 ${BENCH_EXTRA} >> gpurun_out/bench_all.jsonl 2> gpurun_out/bench_${c}_bgram.err || echo "{\"config\": \"$c bgram\", \"failed\": true}" >> gpurun_out/bench_all.jsonl
done
