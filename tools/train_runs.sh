# Training experiments (offline; weights into variants/, reports beside them)
set -x
# fine-tune the depth-6 model on 256^3 frames only
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/train3d.py --depth 6 \
    --init paper_2310_00177_b200/weights/npsd3d_L6.npm --steps 3000 --lr 3e-4 \
    --n 128 --frames 4 --big 12 --big-only --ritz-m 300 --ritz-every 1 --eval256 --seed 71 --out variants/expB13_L6.npm \
    > gpurun_out/r2_trainB13.log 2>&1
cp variants/expB13_L6.* gpurun_out/ 2>/dev/null
