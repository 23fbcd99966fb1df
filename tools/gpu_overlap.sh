D=gpurun_out/${1:-ov}; mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_configs.py -q -x -k "multibatch" > $D/pytest.log 2>&1; echo "pytest exit $?" >> $D/pytest.log
tail -3 $D/pytest.log
bash tools/gpu_env_sweep.sh $1 MCF_DIAG_OVERLAP 0 8 12 16 24
