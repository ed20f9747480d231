export PYTHONUNBUFFERED=1
python tools/psnr_engines.py --cfg cfg2 --dims 256 --batch 65536 --steps 3000 --seeds 6
