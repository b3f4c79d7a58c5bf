timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tests/mp_parity_worker.py > gpurun_out/mp_parity.log 2>&1; echo "rc=$?" >> gpurun_out/mp_parity.log
grep -E "MP-PARITY|rc=|Error|error" gpurun_out/mp_parity.log | head -20
