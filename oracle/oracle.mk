# Builds the CPU CKKS oracle (my restatement; test infrastructure) into oracle/_bin/.
OUT ?= oracle/_bin
CXX := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
$(OUT)/libsf_oracle.so: oracle/ckks_oracle.cpp | $(OUT)
	$(CXX) -std=c++17 -O2 -fopenmp -fPIC -shared -ffp-contract=off -Wall -Wno-unused-function $< -o $@
$(OUT):
	mkdir -p $(OUT)
