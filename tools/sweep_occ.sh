for cfg in "1 2 1" "1 2 2" "0 2 1" "2 2 1"; do set -- $cfg
echo "CAP=$1 FWD=$2 ADJ=$3"; MRF_OCC_CAP=$1 MRF_FWD_CTAS=$2 MRF_ADJ_CTAS=$3 python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1
MRF_OCC_CAP=$1 MRF_FWD_CTAS=$2 MRF_ADJ_CTAS=$3 MRF_LANES=3 python tools/op_breakdown.py --op normal --reps 10 2>&1 | tail -1
done
