for cfg in "1 0" "2 0" "2 10" "2 15" "2 20" "3 10" "3 15" "3 20" "4 15" "4 20"; do
  set -- $cfg
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-roofline --e2e-steps 1 --lanes $1 --lane-tiers $2 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(\"lanes\", d[\"config\"][\"lanes\"], \"tiers\", d[\"config\"][\"lane_tiers\"], round(d[\"value\"]), round(d[\"ms_per_step\"],2))"
done
