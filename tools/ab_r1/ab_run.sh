# Dev A/B: alternate libpgcn builds (PGCN_LIB) on the Reddit-shaped bench step.
#   bash tools/ab_run.sh "<bench args>" lib1 lib2 ...   (lib "-" = the in-tree build)
ARGS=$1; shift
for rep in 1 2; do
  for L in "$@"; do
    if [ "$L" = "-" ]; then unset PGCN_LIB; else export PGCN_LIB=$L; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $ARGS 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); b=d['breakdown']
print('%-34s %7.2f ms/step  ' % ('$L', d['ms_per_step']) + ' '.join('%s %.2f' % (k, v['ms_per_step']) for k, v in b.items() if v['ms_per_step'] > 0.3))"
  done
done
