# Host pipeline chunk-schedule sweep (diagnostics): forward_host at C2 for first-chunk / growth pairs.
for fg in "128 2" "256 2" "128 3" "128 4" "384 2" "512 2" "256 3"; do set -- $fg; echo "first=$1 growth=$2"; DTQ_HOST_FIRST=$1 DTQ_HOST_GROWTH=$2 python tools/xfer_probe.py 2>&1 | grep "forward_host"; done
