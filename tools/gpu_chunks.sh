for c in 2 8 16 32 64; do
  echo "chunks $c $(TS_HYDRO_XFER_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --steps 10 2>&1 | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); e=d["e2e"]; print(round(e["value"]/1e9,4), round(e["sync_value"]/1e9,4))')"
done
