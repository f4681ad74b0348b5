for b in 1 2 3 4; do
  for cfg in c3 c4; do
    TOKENSIM_BPS=$b python bench.py --emulate-ranks 8 --emulate-gs 4,8 --steps 2 --floor-points 1 --config $cfg 2>&1 | tail -1 | python -c "import json,sys; e=json.loads(sys.stdin.read()); print('BPS=$b $cfg', [(c['gpus'], round(c['ms_per_step'],1), c['ranks'][0]['helper_mode'], c['ranks'][0]['grid']) for c in e['curve']])"
  done
done
