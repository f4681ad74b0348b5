# round-end evidence (one GPU): tests, smoke, bench lines, reference arm, emulated scaling
set -x
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_final.txt 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.txt 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c3_final.json 2> gpurun_out/bench_c3_final.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/reference_c3_final.json 2>&1
python bench.py --emulate-ranks 8 --steps 3 > gpurun_out/emulated_scaling_c3_final.json 2>&1
python bench.py --emulate-ranks 8 --steps 3 --config c4 > gpurun_out/emulated_scaling_c4_final.json 2>&1
for c in c1 c2 c4 c6 c7 c8 c9; do python bench.py --config $c --steps 5 --cpu-budget 10 > gpurun_out/bench_${c}_final.json 2>/dev/null; done
python bench.py --config c5 --scaling weak --steps 3 --cpu-budget 10 > gpurun_out/bench_c5_final.json 2>/dev/null
echo done
