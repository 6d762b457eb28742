# Training experiments (offline; weights into variants/, reports beside them)
set -x
python tools/train3d.py --init random --steps 16000 --lr 1e-3 --n 64 --frames 32 --big 16 --ritz-m 400 --ritz-every 1 \
    --eval256 --seed 21 --out variants/expB5.npm > gpurun_out/r2_trainB5.log 2>&1
python tools/train3d.py --init random --steps 8000 --lr 1e-3 --n 128 --frames 16 --big 6 --ritz-m 300 --ritz-every 1 \
    --eval256 --seed 22 --out variants/expB6.npm > gpurun_out/r2_trainB6.log 2>&1
cp variants/expB5.* variants/expB6.* gpurun_out/ 2>/dev/null
