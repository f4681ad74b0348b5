# helper-kernel A/B: C4 / C3 longest points alone, C2, C4 subsets, C3 / C4 at 8 emulated GPUs
A=${1:-ab/libLH.so}; B=${2:-paper_2503_08415_b200/libtokensim.so}
for L in $A $B; do
  echo "== $L"
  TOKENSIM_LIB=$PWD/$L python tools/prof_run.py --config c4 --only 1543 --reps 2 2>&1 | grep "sim ms" | tail -1
  TOKENSIM_LIB=$PWD/$L python tools/prof_run.py --config c3 --only 4596 --reps 2 2>&1 | grep "sim ms" | tail -1
done
python tools/ab.py $A $B --configs c2,c4s4,c4s8 --reps 3 2>&1 | grep -v "^{"
for L in $A $B; do
  TOKENSIM_LIB=$PWD/$L python bench.py --emulate-ranks 8 --emulate-gs 4,8 --steps 2 --floor-points 1 2>&1 | tail -1 | python -c "import json,sys; e=json.loads(sys.stdin.read()); print('$L c3', [(c['gpus'], round(c['ms_per_step'],1), c['ranks'][0]['helper_mode']) for c in e['curve']], 'floor', round(e['chain_floor']['ms'],1))"
  TOKENSIM_LIB=$PWD/$L python bench.py --emulate-ranks 8 --emulate-gs 4,8 --steps 2 --floor-points 1 --config c4 2>&1 | tail -1 | python -c "import json,sys; e=json.loads(sys.stdin.read()); print('$L c4', [(c['gpus'], round(c['ms_per_step'],1), c['ranks'][0]['helper_mode']) for c in e['curve']], 'floor', round(e['chain_floor']['ms'],1))"
done
