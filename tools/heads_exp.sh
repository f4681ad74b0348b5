for cfg in c4 c3; do
  python bench.py --emulate-ranks 8 --steps 2 --config $cfg --floor-points 1 > gpurun_out/heads_${cfg}_auto.log 2>&1
  for K in 0 8 24 48 74; do
    TOKENSIM_HEADS=$K python bench.py --emulate-ranks 8 --emulate-gs 1,8 --steps 2 --config $cfg --floor-points 1 > gpurun_out/heads_${cfg}_$K.log 2>&1
  done
done
python tools/alu_peak.py > gpurun_out/alu.log 2>&1; cp profiles/r2/alu_peak.json gpurun_out/
echo done
