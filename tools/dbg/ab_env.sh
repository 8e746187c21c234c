# A/B an environment variable: bash tools/dbg/ab_env.sh VAR
for v in unset set; do
  if [ $v = set ]; then export $1=1; else unset $1; fi
  echo $1=$v $(timeout 200 python tools/time_pb.py --csr-only 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['csr']; print(round(d['pass_ms']*1e3,1), round(d['iteration_ms']*1e3,1))")
done
