for t in 300000 600000 1000000 100000000000; do BLFMM_NEAR_SPLIT=$t python tools/time_step.py --steps 20 --tag split$t; done > gpurun_out/log.txt 2>&1
for t in 600000 1000000; do echo "split $t"; BLFMM_NEAR_SPLIT=$t timeout 1500 python tools/shard_time.py --worlds 8; done >> gpurun_out/log.txt 2>&1
