# host-landing decode: first call in a fresh process (pinned staging allocation included) per
# slab size / host-copy threads
export PYTHONUNBUFFERED=1
for cfg in "64 4" "64 16" "16 16" "8 16" "32 16" "16 8"; do
set -- $cfg
echo "slab ${1} MB, threads ${2}:"; NVOL_DECODE_SLAB_MB=$1 timeout 300 python tools/decode_e2e.py $2 $2 2>&1 | grep to_host
done
