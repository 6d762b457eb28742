# Training experiments (offline; weights into variants/, reports beside them)
set -x
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --init variants/expB6.npm --steps 5000 --lr 3e-4 --n 128 --frames 16 --big 10 --ritz-m 400 \
    --ritz-every 1 --eval256 --seed 31 --out variants/expB7.npm > gpurun_out/r2_trainB7.log 2>&1
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --init random --steps 14000 --lr 1e-3 --n 128 --frames 20 --big 10 --ritz-m 400 --ritz-every 1 \
    --eval256 --seed 32 --out variants/expB8.npm > gpurun_out/r2_trainB8.log 2>&1
cp variants/expB7.* variants/expB8.* gpurun_out/ 2>/dev/null
