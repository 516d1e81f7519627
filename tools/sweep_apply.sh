cd $GRAFT_REPO_ROOT
for nd in 3 4 5; do
 for sms in 64 80 96 112 0; do
  AMGF_SPMV_SMS=$sms AMGF_TIME_CONFIG="{\"nd_levels\": $nd}" python tools/time_apply.py 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($nd, $sms, round(d['apply_us'],1), round(d['vcycle_us'],1))"
 done
done
