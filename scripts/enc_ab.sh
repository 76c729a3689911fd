# A/B of encoder-attention launch variants: MNMT_ENC_MODE (bucket edges) x MNMT_ENC_QMAX
for cfg in "0 0" "0 1000" "1 0" "1 32" "2 0" "2 16" "2 32" "3 0" "3 32" "3 64" "3 1000"; do
  set -- $cfg
  echo -n "mode $1 qmax $2: "; MNMT_ENC_MODE=$1 MNMT_ENC_QMAX=$2 python scripts/encoder_profile.py 2>&1 | head -1
done
