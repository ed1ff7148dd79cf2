# staged pageable upload, 1 GiB (tools/prof_h2d.py): chunk size x staging buffers.  (A variant that filled every
# chunk with 2-8 pool tasks -- all threads on the earliest chunk first -- measured the same 24.1-24.6 ms and was
# not kept: profiles/r02_h2d_staging.txt.)
for bufs in 4 8 12; do for mb in 16 32 64; do
  CTP_STAGE_BUFS=$bufs CTP_STAGE_CHUNK_MB=$mb python tools/prof_h2d.py 2>&1 | grep "h2d 1 GiB"
done; done
