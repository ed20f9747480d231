export PYTHONUNBUFFERED=1
cd tools/refshim/_tests
for eng in tc simt; do for i in 1 2 3 4 5 6; do
  if [ $eng = simt ]; then export NVOL_TRAIN_ENGINE=simt; else unset NVOL_TRAIN_ENGINE; fi
  PYTHONPATH=../:../../..:$PYTHONPATH timeout 900 python -m pytest test_acceptance.py -q -s -p refshim_adapter -p no:cacheprovider -k "test_7" 2>&1 | grep "^\[PASS\]\|^\[FAIL\]" | sed "s/^/$eng /" | cut -c1-170
done; done
