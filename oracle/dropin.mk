# TEST INFRASTRUCTURE: the drop-in proof (Option A).
# Links the reference's OWN acceptance harness
# (proj/tests/acceptance/acceptance_main.cpp) twice, straight from the
# reference's sources:
#   _ref/acceptance_ref   with the reference's decompiler.cpp (CPU, as shipped)
#   _ref/acceptance_b200  with decompiler.cpp replaced by
#                         integration/ocldec_b200_dropin.cpp, i.e. every
#                         decompile_listing call runs on the GPU through
#                         libocldec_b200.so; all other reference objects are
#                         unchanged.
#   _ref/cfg_check_b200   oracle/cfg_check.cpp with the same drop-in: the
#                         GPU's DecompiledKernel::cfg vs the reference's own
#                         flow graph, field by field.
#   make -C oracle -f dropin.mk    (needs /root/reference: this container only;
#   the binaries travel to the GPU box in oracle/_ref/)
REF      ?= /root/reference/proj
OUT      := _ref
CXX      := /usr/bin/g++
CXXFLAGS := -std=c++20 -O3 -DNDEBUG -fPIC -w -include cstdint \
            -I$(REF)/core/include -I$(REF)/tests/support
CORE     := abi_model asm_frontend builtin_detector cfg codegen diagnostics \
            expr lower oracle structurizer sym_state type_recovery
CORE_O   := $(addprefix $(OUT)/core_,$(addsuffix .o,$(CORE)))
SUP_O    := $(addprefix $(OUT)/sup_,$(addsuffix .o,corpus nestgen grammar envgen))
LIBDIR   := ../paper_2107_07809_b200

all: $(OUT)/acceptance_ref $(OUT)/acceptance_b200 $(OUT)/cfg_check_b200

$(OUT)/core_%.o: $(REF)/core/src/%.cpp
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(OUT)/sup_%.o: $(REF)/tests/support/%.cpp
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(OUT)/acc_main.o: $(REF)/tests/acceptance/acceptance_main.cpp
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(OUT)/dropin_shim.o: ../integration/ocldec_b200_dropin.cpp ../include/ocldec_b200.h
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -I../include -c -o $@ $<

$(OUT)/acceptance_ref: $(OUT)/acc_main.o $(CORE_O) $(OUT)/core_decompiler.o $(SUP_O)
	$(CXX) -o $@ $^ -lpthread

$(OUT)/acceptance_b200: $(OUT)/acc_main.o $(CORE_O) $(OUT)/dropin_shim.o $(SUP_O) $(LIBDIR)/libocldec_b200.so
	$(CXX) -o $@ $(OUT)/acc_main.o $(CORE_O) $(OUT)/dropin_shim.o $(SUP_O) \
	    -L$(LIBDIR) -locldec_b200 -Wl,-rpath,'$$ORIGIN/../../paper_2107_07809_b200' -lpthread -ldl -lrt

# DecompiledKernel::cfg from the drop-in vs the reference's own flow graph
$(OUT)/cfg_check.o: cfg_check.cpp
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(OUT)/cfg_check_b200: $(OUT)/cfg_check.o $(CORE_O) $(OUT)/dropin_shim.o $(LIBDIR)/libocldec_b200.so
	$(CXX) -o $@ $(OUT)/cfg_check.o $(CORE_O) $(OUT)/dropin_shim.o \
	    -L$(LIBDIR) -locldec_b200 -Wl,-rpath,'$$ORIGIN/../../paper_2107_07809_b200' -lpthread -ldl -lrt

.PHONY: all
