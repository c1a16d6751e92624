# e2e (pcbz_judge_host) under host-pipeline knob combinations, C2
#   bash tools/e2e_sweep.sh ["ENV=.. ENV=.." ...]     (default: the list below)
run() { echo "$1 $(env $1 python bench.py --steps 5 --warmup 3 --no-pipeline --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['e2e']['value'],2))")"; }
if [ $# -gt 0 ]; then
  for cfg in "$@"; do run "$cfg"; done
  exit 0
fi
run "X=0"
run "PCBZ_HOST_RAMP=2 PCBZ_HOST_RAMP_DOWN=2 PCBZ_HOST_HEAD=2 PCBZ_HOST_TAIL=2 PCBZ_HOST_EDGE_S=4"
run "PCBZ_HOST_RAMP=2 PCBZ_HOST_RAMP_DOWN=2 PCBZ_HOST_HEAD=1 PCBZ_HOST_TAIL=1 PCBZ_HOST_EDGE_S=4"
run "PCBZ_HOST_RAMP=4 PCBZ_HOST_RAMP_DOWN=4 PCBZ_HOST_HEAD=2 PCBZ_HOST_TAIL=2 PCBZ_HOST_EDGE_S=2"
run "PCBZ_HOST_RAMP_DOWN=2 PCBZ_HOST_TAIL=3 PCBZ_HOST_EDGE_S=4"
run "PCBZ_HOST_RAMP=2 PCBZ_HOST_HEAD=2 PCBZ_HOST_EDGE_S=4"
run "PCBZ_HOST_CHUNK=6"
run "PCBZ_HOST_CHUNK=6 PCBZ_HOST_STREAMS=3"
run "X=0"
