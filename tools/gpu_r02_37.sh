export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python tools/cosched.py --config c3 --levels auto --tunes "nf=0;nf=1;nf=2" --steps 50 2>&1 | grep levels | cut -c1-130
timeout 600 python tools/cosched.py --config c4 --levels auto --tunes "nf=0;nf=1;nf=2" --steps 50 2>&1 | grep levels | cut -c1-130
timeout 900 python tools/cosched.py --config c5 --levels auto --tunes "nf=0;nf=1;nf=2" --steps 15 2>&1 | grep levels | cut -c1-130
