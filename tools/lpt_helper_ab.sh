for v in 0 1 2; do
  for cfg in c3 c4; do
    TOKENSIM_LPT_HELPER=$v python bench.py --emulate-ranks 8 --emulate-gs 8 --steps 3 --floor-points 1 --config $cfg 2>&1 | tail -1 | python -c "import json,sys; e=json.loads(sys.stdin.read()); print('LPT_HELPER=$v $cfg', [(c['gpus'], round(c['ms_per_step'],1), c['ranks'][0]['helper_mode']) for c in e['curve']])"
  done
done
