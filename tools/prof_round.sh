set -x
mkdir -p gpurun_out
python tools/prof_c3.py fwd 2 > /dev/null 2>&1 || exit 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launch_e.csv python tools/prof_c3.py fwd 8 > gpurun_out/c3_launch_e.log 2>&1
ncu --set full --import-source on --clock-control none -s 60 -c 16 -o gpurun_out/c3_full_e -f python tools/prof_c3.py fwd 3 > gpurun_out/c3_full_e.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launch_e.csv python tools/prof_c4.py 3 > gpurun_out/c4_launch_e.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_raster -s 2 -c 2 -o gpurun_out/c4_full_e -f python tools/prof_c4.py 2 > gpurun_out/c4_full_e.log 2>&1
ls -la gpurun_out/*_e*
