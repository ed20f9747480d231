export PYTHONUNBUFFERED=1
cd tools/refshim/_tests
for i in 1 2 3; do PYTHONPATH=../:../../..:$PYTHONPATH timeout 900 python -m pytest test_acceptance.py -q -s -p refshim_adapter -p no:cacheprovider -k "test_7 or test_4" 2>&1 | grep "\[PASS\]\|\[FAIL\]" | cut -c1-200; done
