# c4 near tile DRAM traffic with a minimal metric set (few replays), twice, to check the
# spread between captures.
mkdir -p gpurun_out
python tools/profile_step.py c4 --reps 1 > /dev/null 2>&1
for i in 1 2; do
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_atom.sum \
  --clock-control none -k regex:near_sym -c 1 python tools/profile_step.py c4 --reps 1 2>&1 | grep -E "dram__|lts__|gpu__time" 
done
echo "-- cache-control none"
ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
  --clock-control none -k regex:near_sym -c 1 python tools/profile_step.py c4 --reps 1 2>&1 | grep -E "dram__|lts__|gpu__time"
