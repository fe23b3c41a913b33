export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python tools/cosched.py --config c4 --levels 015152,015652,065652 --tunes "graphs=1" --steps 50 2>&1 | grep levels | cut -c1-110
timeout 600 python tools/cosched.py --config c2 --levels 01102,01602,06602 --tunes "graphs=1" --steps 100 2>&1 | grep levels | cut -c1-110
timeout 900 python tools/cosched.py --config c5 --levels 0151152,0156652,0151652,0156152 --tunes "graphs=1" --steps 15 2>&1 | grep levels | cut -c1-110
