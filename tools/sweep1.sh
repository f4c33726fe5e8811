set -u
mkdir -p gpurun_out
{
echo "== C3 splits"; tools/sweep.sh C3 2 1 2 4
echo "== C2 gb16 splits"; TTS_GROUP_BEAMS=16 tools/sweep.sh C2 8 1 2 4
echo "== C2 gb8 splits"; TTS_GROUP_BEAMS=8 tools/sweep.sh C2 8 1 2
echo "== C2 default"; tools/sweep.sh C2 8 1
echo "== C3 gb8"; TTS_GROUP_BEAMS=8 tools/sweep.sh C3 2 1
} > gpurun_out/sweep1.txt 2>&1
