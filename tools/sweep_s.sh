# E/F occupancy sweep (row-pattern variants); run on the GPU box
V='[{"engine":"fused-f","PIPECG_B200_BPS":2},{"engine":"fused-f","PIPECG_B200_BPS":3},{"engine":"fused-f","PIPECG_B200_BPS":4},{"engine":"fused-e","PIPECG_B200_BPS":2},{"engine":"fused-e","PIPECG_B200_BPS":3}]'
timeout 400 python tools/sweep.py 3d27 400 "$V" 2>&1 | tail -5
timeout 300 python tools/sweep.py 3d7 256 "$V" 2>&1 | tail -5
