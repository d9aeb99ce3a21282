# Recipe: compile the reference's own hot-path sources and tests, unmodified,
# from where they lie under /root/reference, into oracle/_ref/ (git-ignored,
# NOT gpurun-ignored). TEST INFRASTRUCTURE: oracle/_ref is the checker and the
# `--impl reference` CPU arm, never the product.
#   make -f oracle/ref.mk            -> libslotforge_ref.so + 5 test binaries + golden dumper
#   make -f oracle/ref.mk check      -> runs the reference's own tests
REF      ?= /root/reference/proj
OUT      ?= oracle/_ref
JSON_INC ?= $(shell python3 -c "import os,sys; p=os.path.join(sys.prefix,'lib','python%d.%d'%sys.version_info[:2],'site-packages','include','cudnn_frontend','thirdparty'); print(p)")
CXX      ?= g++
CXXFLAGS ?= -std=c++20 -O2 -fPIC -ffp-contract=off -w
INC      := -I$(REF)/include -Ioracle/shim -I$(JSON_INC)
SRCS     := engine layouts vmm kv_attention nonlinear placement harness
OBJS     := $(SRCS:%=$(OUT)/%.o)
TESTS    := test_engine test_layouts test_vmm test_kv test_harness test_nonlinear test_placement

all: $(OUT)/libslotforge_ref.so $(TESTS:%=$(OUT)/%) $(OUT)/ref_golden $(OUT)/ref_bench $(OUT)/ref_on_b200

$(OUT)/%.o: $(REF)/src/%.cpp oracle/shim/Eigen/Dense | $(OUT)
	$(CXX) $(CXXFLAGS) $(INC) -c $< -o $@

$(OUT)/libslotforge_ref.so: $(OBJS)
	$(CXX) -shared -o $@ $^

$(OUT)/test_%: $(REF)/tests/test_%.cpp $(OBJS) oracle/shim/doctest.h
	$(CXX) $(CXXFLAGS) $(INC) $< $(OBJS) -o $@

$(OUT)/ref_golden: oracle/ref_golden.cpp $(OBJS)
	$(CXX) $(CXXFLAGS) $(INC) $< $(OBJS) -o $@

$(OUT)/ref_bench: oracle/ref_bench.cpp $(OBJS)
	$(CXX) $(CXXFLAGS) $(INC) $< $(OBJS) -o $@

# the reference's own hot path on the B200 binding (integration/b200_backend.cpp,
# the reference-side slotforge::Backend over include/sf_b200.h) beside SimBackend
# and the CPU CKKS twin; needs the product library and the oracle library built
$(OUT)/ref_on_b200: oracle/ref_on_b200.cpp oracle/twin_backend.hpp integration/b200_backend.cpp \
		integration/b200_backend.hpp include/sf_b200.h $(OBJS) paper_2602_11470_b200/libsf_b200.so oracle/_bin/libsf_oracle.so
	$(CXX) $(CXXFLAGS) $(INC) -Iinclude oracle/ref_on_b200.cpp integration/b200_backend.cpp $(OBJS) \
		-Lpaper_2602_11470_b200 -lsf_b200 -Loracle/_bin -lsf_oracle \
		-Wl,-rpath,'$$ORIGIN/../../paper_2602_11470_b200:$$ORIGIN/../_bin' -o $@

$(OUT):
	mkdir -p $(OUT)

check: all
	@for t in $(TESTS); do echo "== $$t"; ./$(OUT)/$$t || exit 1; done

.PHONY: all check
