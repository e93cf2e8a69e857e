cd ab/r1 && NCU=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file ../../gpurun_out/ncu_old.csv python tools/acc_probe.py 8 > /dev/null 2>&1; cd ../..
NCU=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_new.csv python tools/acc_probe.py 8 > /dev/null 2>&1
