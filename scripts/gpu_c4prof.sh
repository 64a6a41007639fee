cd _ab/old && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 3 -c 1 -o ../../gpurun_out/m_c4_old python scripts/bench_configs.py c4 > ../../gpurun_out/m_old.log 2>&1; cd ../..
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_brick -s 3 -c 1 -o gpurun_out/m_c4_new python scripts/bench_configs.py c4 > gpurun_out/m_new.log 2>&1
echo done
