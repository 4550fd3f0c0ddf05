# Tile geometry sweep: bench lines (no CPU / e2e) for a workload under tuning env settings.
run() { python bench.py --workload $1 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['fwd_gbs']), round(d.get('bwd_gbs',0)), d['plan'])"; }
for j in 1 2 4 8; do for st in 3 4 6; do SCAN2D_FWD_J=$j SCAN2D_FWD_STAGES=$st run cfg2 "fJ=$j fS=$st"; done; done
for j in 1 2 4; do for st in 2 3 4; do for k in 4 8 16; do SCAN2D_BWD_J=$j SCAN2D_BWD_STAGES=$st SCAN2D_BAND_ROWS=$k run cfg2 "bJ=$j bS=$st K=$k"; done; done; done
for j in 2 4 8; do SCAN2D_FWD_J=$j run cfg3 "fJ=$j"; done
for j in 1 2 4; do SCAN2D_BWD_J=$j run cfg3 "bJ=$j"; done
for j in 2 4 8; do SCAN2D_FWD_J=$j run cfg5 "fJ=$j"; done
