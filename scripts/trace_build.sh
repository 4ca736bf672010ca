# build paper_1805_06557_b200/libswx_trace.so (per-CTA phase marks) next to the default library
set -e
cp paper_1805_06557_b200/libswx.so /tmp/libswx_main.so
python -m paper_1805_06557_b200.build --trace > /dev/null 2>&1
mv paper_1805_06557_b200/libswx.so paper_1805_06557_b200/libswx_trace.so
cp /tmp/libswx_main.so paper_1805_06557_b200/libswx.so
