# usage: bash tools/mana_sweep.sh "N count PLAN|- [G2|U]" ...   (PLAN = L,H,S; U = unstaged kernels)
for cfg in "$@"; do
  set -- $cfg
  if [ "$3" != "-" ]; then export SRE_MANA_PLAN=$3; else unset SRE_MANA_PLAN; fi
  if [ "$4" = "G2" ]; then export SRE_MANA_G2=1; else unset SRE_MANA_G2; fi
  if [ "$4" = "U" ]; then export SRE_MANA_UNSTAGED=1; else unset SRE_MANA_UNSTAGED; fi
  echo -n "$cfg : "; PYTHONPATH=. timeout 120 python tools/mana_rate.py $1 $2 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['prof']; n=p['pass_a']['launched'] or 1; print('%.3g pts/s  A %.1f us  B %.1f us (per launch, %d launches)' % (d['points_per_s'], p['pass_a']['ms_sum']*1e3/n, p['pass_b']['ms_sum']*1e3/n, n))"
done
