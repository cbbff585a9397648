# A/B of accumulate variants on the C2 headline (bench.py), alternating to cancel drift
for i in 1 2; do
  for v in "ENSI_X=0" "ENSI_TC_LOCKSTEP=1" "ENSI_TC_LOCKSTEP=0"; do
    k=0; [ "$v" != "ENSI_X=0" ] && k=4
    echo -n "[$v k=$k] "; env $v timeout 300 python bench.py --no-cpu --no-e2e --no-rot --steps 10 --kernel $k 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['gpu_launches'])"
  done
done
