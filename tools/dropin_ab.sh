# A/B of drop-in host-side variants: alternating runs of the unchanged train_reconstruction
# (tests/cpp/dropin_train.cpp), view-steps/s per run. Usage: bash tools/dropin_ab.sh "ENV_A" "ENV_B" [reps]
A="$1"; B="$2"; R="${3:-3}"
for i in $(seq 1 "$R"); do
  for v in "$A" "$B"; do
    r=$(env $v timeout 300 oracle/_ref/dropin_train_b200 200000 256 75 512 1 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["view_steps_per_s"])')
    echo "$v $r"
  done
done
