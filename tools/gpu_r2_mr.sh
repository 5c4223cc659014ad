# multi-rank bench path on ONE GPU (gloo collectives, 2 ranks sharing cuda:0): functional test
timeout 300 python bench.py --gpus 2 --dist-backend gloo --steps 200 --warmup 5 --no-extra 2>&1 | tail -3 > gpurun_out/mr_weak.log
timeout 300 python bench.py --gpus 2 --dist-backend gloo --scaling strong --steps 50 --warmup 5 --no-extra 2>&1 | tail -3 > gpurun_out/mr_strong.log
timeout 300 python bench.py --gpus 2 --dist-backend gloo --workload L14 --batch 8 --scaling strong --steps 10 --warmup 3 --no-extra 2>&1 | tail -3 > gpurun_out/mr_strong_l14.log
