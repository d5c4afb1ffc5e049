# Bisect the allocation whose uninitialised contents break a solve (KOT_POISON_RANGE).
export KOT_TRD_GRID=48
SEED=${SEED:-0}; IT=${IT:-20}
ref=$(timeout 60 python tools/member_probe.py $SEED $IT 2>&1 | tail -1 | cut -d' ' -f3-8)
echo "ref: $ref"
total=$(KOT_ALLOC_LOG=1 timeout 60 python tools/member_probe.py $SEED $IT 2>&1 | grep -c "kot alloc")
echo "allocations: $total"
ok() { out=$(KOT_POISON=2 KOT_POISON_RANGE=$1:$2 timeout 40 python tools/member_probe.py $SEED $IT 2>&1 | tail -1 | cut -d' ' -f3-8); [ "$out" == "$ref" ]; }
lo=0; hi=$total
if ok $lo $hi; then echo "no failure with full poison"; exit 0; fi
while [ $((hi - lo)) -gt 1 ]; do
  mid=$(( (lo + hi) / 2 ))
  if ! ok $lo $mid; then hi=$mid; elif ! ok $mid $hi; then lo=$mid; else echo "needs both halves [$lo,$mid) [$mid,$hi)"; break; fi
  echo "  -> [$lo, $hi)"
done
echo "culprit range [$lo, $hi)"
KOT_ALLOC_LOG=1 timeout 60 python tools/member_probe.py $SEED $IT 2>&1 | grep "kot alloc" | sed -n "$((lo+1)),$((hi))p" | head
