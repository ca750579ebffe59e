# A/B of the transport line: default library vs variants (build/variants/libb200tally_NAME.so)
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in default "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=build/variants/libb200tally_$v.so; fi
  echo "$v $(BT_LIB_PATH=$lib timeout 300 python tools/transport_line.py --no-reference | python -c 'import json,sys; d=json.load(sys.stdin); print("%.4e"%d["value"], d["events"], d["collisions"])')"
done; done
